#!/bin/bash
cd /root/repo
NCU=/usr/local/cuda/bin/ncu
P="python scripts/profile_kernels.py"
G=tests/golden/plans
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:plan_kernel -s 2 -c 1 \
  -o gpurun_out/prof_plan2pa_b1 -f $P --plan $G/2pa_memory_n8_e64.json --scale 128 --dtype bf16 > /dev/null 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:pull_reduce -s 2 -c 1 \
  -o gpurun_out/prof_2pa_16k -f $P --algo 2pa --bytes 16384 --dtype bf16 > /dev/null 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:plan_kernel -s 2 -c 1 \
  -o gpurun_out/prof_plan1pa_b64 -f $P --plan $G/1pa_n8_e64.json --scale 8192 --dtype bf16 > /dev/null 2>&1
echo done
