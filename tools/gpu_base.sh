# round-2 session-2 baseline: probe cfg1-5, bench line, ncu --set full of the k_wgroup passes (cfg4 full size)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 300 python tools/probe.py 1 2 3 4 5 > gpurun_out/probe.log 2>&1; tail -40 gpurun_out/probe.log
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 600 gpurun_out/bench.json
TAG=${TAG:-base}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wgroup -c 2 -o gpurun_out/prof_$TAG python tools/one_build.py 4 0 1 > gpurun_out/ncu_$TAG.log 2>&1; tail -3 gpurun_out/ncu_$TAG.log
