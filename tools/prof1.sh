#!/bin/bash
# One full ncu capture of a single stage-kernel launch of tools/profile_stage.py
# (default: launch 9 = GTS stage 1 on cfg2), report copied into gpurun_out/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
TAG=${1:-one}; SKIP=${2:-77}
mkdir -p gpurun_out
python tools/profile_stage.py > gpurun_out/prof1_plain_$TAG.log 2>&1 || { echo plain failed; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:stage_cross -s $SKIP -c 1 \
    -o gpurun_out/one_$TAG python tools/profile_stage.py > gpurun_out/ncu1_$TAG.log 2>&1
tail -2 gpurun_out/ncu1_$TAG.log; ls -la gpurun_out/one_$TAG.ncu-rep
