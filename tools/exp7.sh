cd ${GRAFT_REPO_ROOT:-.}
V=$PWD/build/var
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_ranks_gpu.py -q -m gpu -x 2>&1 | tail -5 > gpurun_out/exp7_tests.txt
cat gpurun_out/exp7_tests.txt
bash tools/gpu_var.sh tpc2:default: tpc1:$V/tpc1/libamr.so: tpc3:$V/tpc3/libamr.so: > gpurun_out/exp7.txt 2>&1
cat gpurun_out/exp7.txt
