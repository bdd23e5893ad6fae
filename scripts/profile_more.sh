#!/bin/bash
# ncu evidence for the kernels profile.sh does not cover (K4 two-shot LL, K8
# direct RS, K7 ring AG, K9 ring RS, K1 at C3 sizes) + NVLS probe.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
P="python scripts/profile_kernels.py"
(nvidia-smi -q | grep -i -A6 "fabric\|nvlink\|multicast"; timeout 120 python scripts/nvls_probe.py) > gpurun_out/nvls_probe.txt 2>&1
full() {   # name kernel-regex args...
  local name=$1 k=$2; shift 2
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o gpurun_out/prof_$name -f "$@" > gpurun_out/ncu_$name.log 2>&1
  echo "$name rc=$?"
}
full 2pall_1k ll_twoshot $P --algo 2pa_ll --bytes 1024 --dtype bf16 --iters 3
full 2pall_256k ll_twoshot $P --algo 2pa_ll --bytes 262144 --dtype bf16 --iters 3
full 1pa_256k ll_oneshot $P --algo 1pa --bytes 262144 --dtype bf16 --iters 3
full 1pa_1k ll_oneshot $P --algo 1pa --bytes 1024 --dtype bf16 --iters 3
full rs_256m pull_reduce $P --kind reducescatter --algo rs_direct --bytes 268435456 --dtype bf16 --iters 3
full ringrs_256m ring_kernel $P --kind reducescatter --algo ring_rs --bytes 268435456 --dtype bf16 --iters 3
full ringag_256m ring_gather $P --kind allgather --algo ring_ag --bytes 268435456 --dtype bf16 --iters 3
# K5 control path through the emulated switch (per-rank loads / stores in place of multimem)
full nvlsemul_64m nvls_kernel $P --algo switch_2pa --emulate-nvls --bytes 67108864 --dtype bf16 --iters 3
ls -la gpurun_out/*.ncu-rep
