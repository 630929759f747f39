cd ${GRAFT_REPO_ROOT:-.}
V=$PWD/build/var
bash tools/gpu_var.sh base:default: t128:default:AMR_THREADS=128 minb5:$V/minb5/libamr.so: minb3:$V/minb3/libamr.so: minb3t128:$V/minb3/libamr.so:AMR_THREADS=128 > gpurun_out/exp1.txt 2>&1
AMR_LIB_PATH=$V/probe/libamr.so python tools/phase_probe.py > gpurun_out/probe1.txt 2>&1
cat gpurun_out/exp1.txt gpurun_out/probe1.txt
