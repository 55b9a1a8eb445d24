# session-5: chain-length floor (two tiles per chain); sweep, then the full suite and the bench line
mkdir -p gpurun_out
timeout 900 python tools/sweep.py > gpurun_out/sweep_r02g.jsonl 2> gpurun_out/sweep_r02g.err; echo "sweep rc=$?"
python - <<'PY'
import json
for l in open('gpurun_out/sweep_r02g.jsonl'):
    r=json.loads(l); print(r['sweep'], r['n'], r['levels'], 'wt %.3f wm %.3f' % (r['wt_ms'], r['wm_ms']))
PY
timeout 1100 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/gputest_r02g.log; cat gpurun_out/gputest_r02g.log
timeout 300 python bench.py > gpurun_out/bench_r02g.json 2> gpurun_out/bench_r02g.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/bench_r02g.json
timeout 600 python tools/report_time.py 1 2 3 4 5; cp gpurun_out/report_time.jsonl gpurun_out/report_time_r02g.jsonl
