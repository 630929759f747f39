cd ${GRAFT_REPO_ROOT:-.}
timeout 1500 python tools/cfg5_try.py cfg5 16 > gpurun_out/cfg5_try2.log 2>&1; tail -8 gpurun_out/cfg5_try2.log
bash tools/round2_profile.sh r2b
