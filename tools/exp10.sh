cd ${GRAFT_REPO_ROOT:-.}
timeout 1500 python -m pytest tests/test_octree_gpu.py -q -x -s 2>&1 | tail -25 > gpurun_out/exp10_tests.txt
cat gpurun_out/exp10_tests.txt
nproc; free -g | head -2
