cd ${GRAFT_REPO_ROOT:-.}
timeout 1500 python -m pytest tests/test_devprog_gpu.py -q -x -s 2>&1 | tail -25 > gpurun_out/exp14_devprog.txt
cat gpurun_out/exp14_devprog.txt
timeout 2400 python -m pytest tests -q -x -m gpu 2>&1 | tail -8 > gpurun_out/exp14_all.txt
cat gpurun_out/exp14_all.txt
bash tools/gpu_var.sh final:default: > gpurun_out/exp14.txt 2>&1
cat gpurun_out/exp14.txt
