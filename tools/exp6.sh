cd ${GRAFT_REPO_ROOT:-.}
V=$PWD/build/var
bash tools/gpu_var.sh base:default: ilp:$V/ilp/libamr.so: gu2:$V/gu2/libamr.so: > gpurun_out/exp6.txt 2>&1
cat gpurun_out/exp6.txt
