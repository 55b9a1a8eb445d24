# session-5 experiments: remainder-first level split and four 32-bit records per lane (WT_WG_E32)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1000 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bign.py -x -q 2>&1 | tail -4
TUNE_DIR=tvar timeout 600 python tools/tune.py run 5 2>&1 | tee gpurun_out/tune_e32.log
SWEEP_ONLY=sigma timeout 600 python tools/sweep.py > gpurun_out/sweep_first.jsonl 2> gpurun_out/sweep.err; echo "sweep rc=$?"
SWEEP_ONLY=sigma WT_TAUS_TAIL=1 timeout 600 python tools/sweep.py > gpurun_out/sweep_tail.jsonl 2>> gpurun_out/sweep.err; echo "sweep tail rc=$?"
python - <<'PY'
import json
a=[json.loads(l) for l in open('gpurun_out/sweep_first.jsonl')]
b=[json.loads(l) for l in open('gpurun_out/sweep_tail.jsonl')]
for x,y in zip(a,b): print(x['levels'], 'first %.3f ms  tail %.3f ms  wm %.3f ms' % (x['wt_ms'], y['wt_ms'], x['wm_ms']))
PY
