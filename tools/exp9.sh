cd ${GRAFT_REPO_ROOT:-.}
V=$PWD/build/var
bash tools/gpu_var.sh base:default: rolled:$V/rolled/libamr.so: > gpurun_out/exp9.txt 2>&1
cat gpurun_out/exp9.txt
