#!/bin/bash
# ncu --set full of the compiled plan kernels (C5 b=64) and K13 two-shot (b=256) -> gpurun_out/prof_summary_r2b/
NCU=/usr/local/cuda/bin/ncu
P="python scripts/profile_kernels.py"
G=tests/golden/plans
mkdir -p gpurun_out
rm -f gpurun_out/*.ncu-rep
full() { local name=$1 k=$2; shift 2
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_$name -f "$@" > gpurun_out/ncu_$name.log 2>&1; echo "$name rc=$?"; }
full plan2pa_b64_compiled plan_single $P --plan $G/2pa_memory_n8_e64.json --scale 8192 --dtype bf16 --iters 4
full plan2pall_b64_compiled plan_ll $P --plan $G/2pa_ll_n8_e64.json --scale 8192 --dtype bf16 --iters 4
full plan1pa_b64_compiled plan_ll $P --plan $G/1pa_n8_e64.json --scale 8192 --dtype bf16 --iters 4
full fused_b256 ar_rmsnorm $P --kind fused --algo 2pa --bytes 4194304 --dtype bf16 --iters 3
python scripts/summarize_profiles.py round2b gpurun_out/prof_summary_r2b > /dev/null 2>&1; echo "summary rc=$?"
rm -f gpurun_out/*.ncu-rep
