cd ${GRAFT_REPO_ROOT:-.}
timeout 1200 python -m pytest tests/test_parity_scale.py -q -m gpu -k "cfg4 or cfg3" 2>&1 | tail -4
timeout 2400 python tools/cfg5_try.py cfg5 8 > gpurun_out/cfg5_try.log 2>&1; tail -12 gpurun_out/cfg5_try.log
