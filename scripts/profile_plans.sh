#!/bin/bash
# ncu evidence for the plan interpreter (K10) at C5 shapes and the ring kernels.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
P="python scripts/profile_kernels.py"
G=tests/golden/plans
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:plan_kernel -s 2 -c 1 \
  -o gpurun_out/prof_plan2pa_b1 -f $P --plan $G/2pa_memory_n8_e64.json --scale 128 --dtype bf16 > /dev/null 2>&1
echo "plan2pa b1 rc=$?"
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:plan_kernel -s 2 -c 1 \
  -o gpurun_out/prof_plan2pa_b64 -f $P --plan $G/2pa_memory_n8_e64.json --scale 8192 --dtype bf16 > /dev/null 2>&1
echo "plan2pa b64 rc=$?"
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:plan_kernel -s 2 -c 1 \
  -o gpurun_out/prof_plan1pa_b1 -f $P --plan $G/1pa_n8_e64.json --scale 128 --dtype bf16 > /dev/null 2>&1
echo "plan1pa b1 rc=$?"
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:ring_kernel -s 2 -c 1 \
  -o gpurun_out/prof_ring_2pr_64m -f $P --algo 2pr --bytes 67108864 --dtype bf16 > /dev/null 2>&1
echo "ring rc=$?"
