cd ${GRAFT_REPO_ROOT:-.}
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_parity_scale.py -q -m gpu -x 2>&1 | tail -5 > gpurun_out/exp2_tests.txt
bash tools/gpu_var.sh pers:default: pers444:default:AMR_GRID_CAP=444 > gpurun_out/exp2.txt 2>&1
cat gpurun_out/exp2_tests.txt gpurun_out/exp2.txt
