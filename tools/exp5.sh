cd ${GRAFT_REPO_ROOT:-.}
timeout 1700 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/exp5_tests.txt
cat gpurun_out/exp5_tests.txt
bash tools/gpu_var.sh pdl:default: nopdl:default:AMR_PDL=0 > gpurun_out/exp5.txt 2>&1
cat gpurun_out/exp5.txt
