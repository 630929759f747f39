cd ${GRAFT_REPO_ROOT:-.}
timeout 1500 python -m pytest tests/test_devmesh_gpu.py -q -x -s 2>&1 | tail -25 > gpurun_out/exp12_tests.txt
cat gpurun_out/exp12_tests.txt
# cfg4 oracle fields (host memory: more than the build container has); the golden comes back in gpurun_out/
AMR_GOLDEN_OUT=$PWD/gpurun_out timeout 2400 python tests/golden/make_golden_scale.py fields cfg4 > gpurun_out/gold_cfg4.log 2>&1
tail -5 gpurun_out/gold_cfg4.log; ls -la gpurun_out/scale_cfg4.npz
