#!/bin/bash
# ncu --set full of K13 two-shot at C5 b=64 and b=256 -> gpurun_out/prof_summary_k13/
NCU=/usr/local/cuda/bin/ncu
P="python scripts/profile_kernels.py"
mkdir -p gpurun_out
rm -f gpurun_out/*.ncu-rep
full() { local name=$1 k=$2; shift 2
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_$name -f "$@" > gpurun_out/ncu_$name.log 2>&1; echo "$name rc=$?"; }
full fused_b64 ar_rmsnorm $P --kind fused --algo 2pa --bytes 1048576 --dtype bf16 --iters 3
full fused_b256 ar_rmsnorm $P --kind fused --algo 2pa --bytes 4194304 --dtype bf16 --iters 3
python scripts/summarize_profiles.py k13 gpurun_out/prof_summary_k13 > /dev/null 2>&1; echo "summary rc=$?"
rm -f gpurun_out/*.ncu-rep
