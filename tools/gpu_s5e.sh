# session-5: node tables (A4) and block entries of non-last groups on the side stream; A/B, then the suite and the bench line
mkdir -p gpurun_out
for i in 1 2; do
WT_NO_SIDE_A4=1 timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('main-stream A4: %.4f ms/step' % d['ms_per_step'])"
timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('side-stream A4: %.4f ms/step' % d['ms_per_step'])"
done 2>&1 | tee gpurun_out/side_a4.log
timeout 600 python tools/report_time.py 3 4 5 | tee -a gpurun_out/side_a4.log
timeout 1100 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/gputest_r02h.log; cat gpurun_out/gputest_r02h.log
timeout 300 python bench.py > gpurun_out/bench_r02h.json 2> gpurun_out/bench_r02h.err; echo "bench rc=$?"; tail -c 1200 gpurun_out/bench_r02h.json
