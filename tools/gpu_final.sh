TAG=${TAG:-r02}
mkdir -p gpurun_out
timeout 1100 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/gputest_$TAG.log; cat gpurun_out/gputest_$TAG.log
timeout 900 python tools/sweep.py > gpurun_out/sweep_$TAG.jsonl 2> gpurun_out/sweep_$TAG.err; echo "sweep rc=$?"
bash tools/gpu_report.sh
timeout 300 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; tail -c 2500 gpurun_out/bench_$TAG.json
