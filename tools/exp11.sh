cd ${GRAFT_REPO_ROOT:-.}
timeout 1500 python -m pytest tests/test_api_kernels_gpu.py tests/test_ranks_gpu.py -q -x 2>&1 | tail -8
bash tools/sanitize.sh
