#!/bin/bash
# ncu capture of the stage kernel on cfg2 (tools/profile_stage.py: launches
# 0-3 LTS round start, 4-7 LTS finest-only slice, 8-11 GTS step), each ncu run
# only after the plain command exited 0.  Usage: tools/prof.sh TAG [threads]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
TAG=${1:-p}
export AMR_THREADS=${2:-128}
mkdir -p gpurun_out
python tools/profile_stage.py > gpurun_out/prof_plain_$TAG.log 2>&1 || { echo plain failed; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:stage_cross -s 68 -c 12 \
    -o /tmp/prof_$TAG python tools/profile_stage.py > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log
python tools/ncu_summary.py /tmp/prof_$TAG.ncu-rep > gpurun_out/sum_$TAG.md 2>&1
python tools/ncu_traffic.py /tmp/prof_$TAG.ncu-rep gpurun_out/traffic_$TAG.json > /dev/null 2>&1
python tools/ncu_stalls.py /tmp/prof_$TAG.ncu-rep stage_cross 1 40 > gpurun_out/stalls_${TAG}_lts1.txt 2>&1
python tools/ncu_stalls.py /tmp/prof_$TAG.ncu-rep stage_cross 9 40 > gpurun_out/stalls_${TAG}_gts1.txt 2>&1
cat gpurun_out/sum_$TAG.md
python tools/ncu_lines.py /tmp/prof_$TAG.ncu-rep stage_cross 9 40 > gpurun_out/lines_${TAG}_gts1.txt 2>&1
ncu -i /tmp/prof_$TAG.ncu-rep --page details --launch-skip 9 --launch-count 1 > gpurun_out/details_${TAG}_gts1.txt 2>&1
