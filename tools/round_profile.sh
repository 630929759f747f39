# One GPU call: parity, bench, the bench's ncu launch list, and a full ncu capture
# of the stage kernel (each ncu run only after the same command exited 0).
# Summaries land in gpurun_out/ (copy the ones to keep into profiles/).
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-r1}
K=${KREGEX:-stage_cross}
bash tests/gpu_parity.sh > gpurun_out/parity_$TAG.log 2>&1; grep -E "passed|failed" gpurun_out/parity_$TAG.log | tail -3
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$TAG.log 2>&1; tail -1 gpurun_out/bench_$TAG.log | cut -c1-300
python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/bench_small_$TAG.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
      --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_launches_$TAG.log 2>&1
python tools/profile_stage.py > gpurun_out/prof_plain_$TAG.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"$K" -s 68 -c 12 \
      -o /tmp/prof_$TAG python tools/profile_stage.py > gpurun_out/ncu_$TAG.log 2>&1
tail -1 gpurun_out/ncu_$TAG.log
python tools/ncu_summary.py /tmp/prof_$TAG.ncu-rep > gpurun_out/sum_$TAG.md 2>&1
python tools/ncu_traffic.py /tmp/prof_$TAG.ncu-rep gpurun_out/traffic_$TAG.json > /dev/null 2>&1
for k in 1 9; do python tools/ncu_lines.py /tmp/prof_$TAG.ncu-rep $K $k 30 > gpurun_out/lines_${TAG}_$k.txt 2>&1; done
python tools/ncu_stalls.py /tmp/prof_$TAG.ncu-rep $K 9 20 > gpurun_out/stalls_$TAG.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:"$K" -s 77 -c 1 \
    -o gpurun_out/prof_${TAG}_gts1 python tools/profile_stage.py > /dev/null 2>&1
cat gpurun_out/sum_$TAG.md
