cd ${GRAFT_REPO_ROOT:-.}
V=$PWD/build/var
TPC=1 AMR_LIB_PATH=$V/probe1/libamr.so python tools/phase_probe.py 2>&1 | grep "gts stage" > gpurun_out/probe_tpc1.txt
TPC=2 AMR_LIB_PATH=$V/probe2/libamr.so python tools/phase_probe.py 2>&1 | grep "gts stage" > gpurun_out/probe_tpc2.txt
cat gpurun_out/probe_tpc1.txt gpurun_out/probe_tpc2.txt
