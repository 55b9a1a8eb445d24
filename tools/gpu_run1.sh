set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python tools/probe.py 1 2 3 4 5 > gpurun_out/probe_v3.log 2>&1; tail -60 gpurun_out/probe_v3.log
timeout 120 python tools/one_build.py 4 16777216 2 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_group -c 2 -o gpurun_out/prof_v3 python tools/one_build.py 4 16777216 1 > gpurun_out/ncu_v3.log 2>&1; tail -5 gpurun_out/ncu_v3.log
