# quick GPU check: parity subset + per-kernel probe (argument: extra pytest -k filter)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -15
timeout 300 python tools/probe.py ${PROBE_CFGS:-1 2 3 4} 2>&1 | tail -70
