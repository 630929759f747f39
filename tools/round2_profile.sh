#!/bin/bash
# Round-2 evidence in one GPU call: the GPU test suite, the default bench line
# (+ the reference arm), the bench's ncu launch list, a full ncu capture of the
# stage kernel on cfg2 (stalls, source lines, traffic), and the DRAM traffic of
# the stage kernel on cfg3 / cfg4.  Every ncu run follows a plain run of the
# same command that exited 0.  Summaries land in gpurun_out/.
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-r2}
K=stage_cross
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$TAG.txt
timeout 2400 python -m pytest tests -m gpu -q -rA > gpurun_out/parity_$TAG.log 2>&1; grep -E "passed|failed" gpurun_out/parity_$TAG.log | tail -2
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -c 400 gpurun_out/bench_$TAG.json
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
python bench.py --steps 1 --warmup 1 --no-cpu --side none > gpurun_out/bench_small_$TAG.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
      --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 1 --no-cpu --side none > gpurun_out/ncu_launches_$TAG.log 2>&1
python tools/launch_summary.py gpurun_out/launches_$TAG.csv > gpurun_out/launches_summary_$TAG.md 2>&1
python tools/profile_stage.py > gpurun_out/prof_plain_$TAG.log 2>&1 && \
  ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"$K" \
      -o /tmp/prof_$TAG python tools/profile_stage.py > gpurun_out/ncu_$TAG.log 2>&1
python tools/ncu_summary.py /tmp/prof_$TAG.ncu-rep > gpurun_out/sum_$TAG.md 2>&1
python tools/ncu_traffic.py /tmp/prof_$TAG.ncu-rep gpurun_out/traffic_$TAG.json cfg2 > /dev/null 2>&1
# captured launches (cfg2): LTS round start, all tiles in one launch per stage (0..3), finest-only slice (4..7, lean), GTS step (8..11)
for k in 2 9; do python tools/ncu_lines.py /tmp/prof_$TAG.ncu-rep $K $k 30 > gpurun_out/lines_${TAG}_$k.txt 2>&1; done
python tools/ncu_stalls.py /tmp/prof_$TAG.ncu-rep $K 9 20 > gpurun_out/stalls_$TAG.txt 2>&1
python tools/ncu_stalls.py /tmp/prof_$TAG.ncu-rep $K 2 20 > gpurun_out/stalls_${TAG}_lts.txt 2>&1
cat gpurun_out/sum_$TAG.md
# cfg3, cfg4: the same driver (the profiled launches are bracketed by cudaProfilerStart/Stop)
python tools/profile_stage.py --config cfg3 > gpurun_out/prof_plain_${TAG}_cfg3.log 2>&1 && \
  ncu --set full --clock-control none --profile-from-start off -k regex:"$K" \
      -o /tmp/prof_${TAG}_cfg3 python tools/profile_stage.py --config cfg3 > gpurun_out/ncu_${TAG}_cfg3.log 2>&1
python tools/ncu_summary.py /tmp/prof_${TAG}_cfg3.ncu-rep > gpurun_out/sum_${TAG}_cfg3.md 2>&1
python tools/ncu_traffic.py /tmp/prof_${TAG}_cfg3.ncu-rep gpurun_out/traffic_${TAG}_cfg3.json cfg3 > /dev/null 2>&1
python tools/profile_stage.py --config cfg4 > gpurun_out/prof_plain_${TAG}_cfg4.log 2>&1 && \
  ncu --set full --clock-control none --profile-from-start off -k regex:"$K" \
      -o /tmp/prof_${TAG}_cfg4 python tools/profile_stage.py --config cfg4 > gpurun_out/ncu_${TAG}_cfg4.log 2>&1
python tools/ncu_summary.py /tmp/prof_${TAG}_cfg4.ncu-rep > gpurun_out/sum_${TAG}_cfg4.md 2>&1
python tools/ncu_traffic.py /tmp/prof_${TAG}_cfg4.ncu-rep gpurun_out/traffic_${TAG}_cfg4.json cfg4 > /dev/null 2>&1
cat gpurun_out/traffic_${TAG}*.json
