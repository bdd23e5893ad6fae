#!/bin/bash
# ncu evidence for the dominant kernels (1 GPU, 8 co-resident ranks).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
P="python scripts/profile_kernels.py"
G=tests/golden/plans
# launch list of the bench command itself (cold-cache, serialised; no sweep)
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv -c 400 \
  --log-file gpurun_out/launches_headline.csv python bench.py --steps 2 --warmup 3 --no-sweep > /dev/null 2>&1
echo "launch list rc=$?"
full() {   # name kernel-regex args...
  local name=$1 k=$2; shift 2
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o gpurun_out/prof_$name -f "$@" > gpurun_out/ncu_$name.log 2>&1
  echo "$name rc=$?"
}
full 2pa_256m pull_reduce $P --algo 2pa --bytes 268435456 --dtype bf16 --iters 3
full 2pa_1m pull_reduce $P --algo 2pa --bytes 1048576 --dtype bf16 --iters 3
full 1pa_c1 ll_oneshot $P --algo 1pa --bytes 1048576 --dtype f32 --iters 3
full 2pr_64m ring_kernel $P --algo 2pr --bytes 67108864 --dtype bf16 --iters 3
full ag_256m push_gather $P --kind allgather --algo allpairs_ag --bytes 268435456 --dtype bf16 --iters 3
full fused_b256 ar_rmsnorm $P --kind fused --algo 2pa --bytes 4194304 --dtype bf16 --iters 3
full plan2pa_b1 plan_kernel $P --plan $G/2pa_memory_n8_e64.json --scale 128 --dtype bf16
full plan1pa_b64 plan_kernel $P --plan $G/1pa_n8_e64.json --scale 8192 --dtype bf16
ls -la gpurun_out/*.ncu-rep
