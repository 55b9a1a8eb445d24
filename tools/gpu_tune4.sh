nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bign.py -x -q 2>&1 | tail -1
TUNE_CPW=${TUNE_CPW:-16} timeout 900 python tools/tune.py run ${TUNE_CFGS:-4 5}
