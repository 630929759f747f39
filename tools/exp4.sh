cd ${GRAFT_REPO_ROOT:-.}
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/exp4_tests.txt
cat gpurun_out/exp4_tests.txt
