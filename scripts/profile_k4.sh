#!/bin/bash
# ncu --set full of K4 (LL two-shot) at 1 KiB / 256 KiB / 1 MiB, summarised on the box.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
P="python scripts/profile_kernels.py"
for s in 1024:1k 262144:256k 1048576:1m; do
  timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:ll_twoshot -s 2 -c 1 \
    -o gpurun_out/prof_2pall_${s#*:} -f $P --algo 2pa_ll --bytes ${s%%:*} --dtype bf16 --iters 3 \
    > gpurun_out/ncu_2pall_${s#*:}.log 2>&1
  echo "2pall_${s#*:} rc=$?"
done
python scripts/summarize_profiles.py k4 gpurun_out/prof_k4 > /dev/null 2>&1; echo "summary rc=$?"
rm -f gpurun_out/*.ncu-rep
