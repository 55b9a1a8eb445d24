# parity subset, probe, then an ncu --set full capture of the group kernels (cfg4 prefix)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -5
timeout 300 python tools/probe.py ${PROBE_CFGS:-1 2 3 4} 2>&1 | tail -70
TAG=${TAG:-x}
timeout 120 python tools/one_build.py 4 16777216 2 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_group -c 2 -o gpurun_out/prof_$TAG python tools/one_build.py 4 16777216 1 > gpurun_out/ncu_$TAG.log 2>&1; tail -3 gpurun_out/ncu_$TAG.log
