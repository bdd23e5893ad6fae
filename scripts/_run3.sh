set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_multiprocess.py -x -q 2>&1 | tail -3
for a in "" 1pa_hb 2pa; do ALGO=$a timeout 120 python scripts/fused_probe.py; done
CF_LIB_PATH=$PWD/paper_2504_09014_b200/libcf_ts.so PLANS=2pa_memory_n8_e64,2pa_ll_n8_e64,1pa_n8_e64 ALGOS=2pa,2pa_ll,1pa SIZES=16384 timeout 300 python scripts/ts_probe.py > gpurun_out/ts_plans.log 2>&1; echo ts rc=$?
timeout 300 python scripts/c5_ab.py
