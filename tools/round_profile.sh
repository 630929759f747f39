# One GPU call: parity, bench, the bench's ncu launch list, and a full ncu capture
# of the stage kernel (each ncu run only after the same command exited 0).
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-r1}
bash tests/gpu_parity.sh > gpurun_out/parity_$TAG.log 2>&1; grep -E "passed|failed" gpurun_out/parity_$TAG.log | tail -3
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$TAG.log 2>&1; tail -1 gpurun_out/bench_$TAG.log
python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/bench_small_$TAG.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
      --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_launches_$TAG.log 2>&1
python tools/profile_stage.py > gpurun_out/prof_plain_$TAG.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"stage_kernel" -s 68 -c 12 \
      -o gpurun_out/prof_$TAG python tools/profile_stage.py > gpurun_out/ncu_$TAG.log 2>&1
tail -1 gpurun_out/ncu_$TAG.log
