#!/bin/bash
# One gpurun call: bench (JSON line), ncu launch list + full captures of every
# kernel, summarised ON THE BOX into gpurun_out/prof_summary/ (the .ncu-rep
# files are deleted afterwards so gpurun_out stays under the 64 MiB return cap;
# the two headline reports are kept).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
bash scripts/profile.sh
bash scripts/profile_more.sh
python scripts/summarize_profiles.py round1 gpurun_out/prof_summary > /dev/null 2>&1; echo "summary rc=$?"
mkdir -p gpurun_out/keep
mv gpurun_out/prof_2pa_256m.ncu-rep gpurun_out/keep/ 2>/dev/null
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out
