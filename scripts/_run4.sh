mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | tail -2
L=$PWD/paper_2504_09014_b200/libcf_ts.so
CF_LIB_PATH=$L BATCH=16,64 ALGO=2pa timeout 120 python scripts/k13_ts.py 2>&1 | grep -E "^---|rank 0 " 
for a in 2pa 1pa_hb; do for t in 256 512; do echo "$a threads $t"; CF_K13_THREADS=$t ALGO=$a timeout 120 python scripts/fused_probe.py; done; done
echo default; timeout 120 python scripts/fused_probe.py
