nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
TUNE_CPW=${TUNE_CPW:-8,16} timeout 900 python tools/tune.py run ${TUNE_CFGS:-3 4}
