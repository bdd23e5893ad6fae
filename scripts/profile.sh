#!/bin/bash
# ncu evidence for the dominant kernels (1 GPU, 8 co-resident ranks).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
P="python scripts/profile_kernels.py"
# launch list of the headline bench configuration (cold-cache, serialised)
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_headline.csv $P --algo 2pa --bytes 268435456 --dtype bf16 --iters 5 > /dev/null 2>&1
echo "launch list rc=$?"
# full sets: headline two-shot, C1 one-shot LL, 1 MiB two-shot, C5 plan
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:pull_reduce -s 2 -c 1 \
  -o gpurun_out/prof_2pa_256m -f $P --algo 2pa --bytes 268435456 --dtype bf16 --iters 3 > gpurun_out/ncu_2pa.log 2>&1
echo "2pa rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:ll_oneshot -s 2 -c 1 \
  -o gpurun_out/prof_1pa_c1 -f $P --algo 1pa --bytes 1048576 --dtype f32 --iters 3 > gpurun_out/ncu_1pa.log 2>&1
echo "1pa rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:pull_reduce -s 2 -c 1 \
  -o gpurun_out/prof_2pa_1m -f $P --algo 2pa --bytes 1048576 --dtype bf16 --iters 3 > gpurun_out/ncu_2pa1m.log 2>&1
echo "2pa1m rc=$?"
ls -la gpurun_out/
