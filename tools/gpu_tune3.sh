nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
for v in ns_t16_3k ns_t16_6k; do WT_LIB_PATH=tune_variants/lib_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "config or random" 2>&1 | tail -1; done
TUNE_CPW=${TUNE_CPW:-16} timeout 900 python tools/tune.py run ${TUNE_CFGS:-4 5}
