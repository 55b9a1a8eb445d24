# session-5: 7 CTAs per SM for the 8-bit pass (smaller unstaged tiles; 64-bit word-rank entries, WT_WG_RP64)
mkdir -p gpurun_out
WT_LIB_PATH=tvar/lib_rp64.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "config or random or remainder or adversarial or zipf" 2>&1 | tail -2
TUNE_DIR=tvar timeout 900 python tools/tune.py run 4 3 5 2>&1 | tee gpurun_out/tune_cta7.log
