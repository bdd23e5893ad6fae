#!/bin/bash
# Round-2 ncu evidence (1 GPU, 8 co-resident ranks): launch list of the bench
# command, --set full of the headline kernel and of the kernels round 2
# changed, summarised on the box into gpurun_out/prof_summary_r2/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rm -f gpurun_out/*.ncu-rep gpurun_out/launches*.csv
NCU=/usr/local/cuda/bin/ncu
P="python scripts/profile_kernels.py"
G=tests/golden/plans
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
full 2pr_256m pull_reduce $P --algo 2pr --bytes 268435456 --dtype bf16 --iters 3
full ag_bulk_256m push_gather_bulk $P --kind allgather --algo allpairs_ag --bytes 268435456 --dtype bf16 --iters 3
full rs_ring_order_256m pull_reduce $P --kind reducescatter --algo ring_rs --bytes 268435456 --dtype bf16 --iters 3
full fused_b64 ar_rmsnorm $P --kind fused --algo 2pa --bytes 1048576 --dtype bf16 --iters 3
full plan2pa_b1 plan_kernel $P --plan $G/2pa_memory_n8_e64.json --scale 128 --dtype bf16 --iters 4
python scripts/summarize_profiles.py round2 gpurun_out/prof_summary_r2 > /dev/null 2>&1; echo "summary rc=$?"
rm -f gpurun_out/*.ncu-rep
python scripts/write_peak.py
