#!/bin/bash
# kernel-3 bring-up: parity tests, then cfg2 bench lines for kernel 3 (128/256 threads)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/k3_smi.txt
for t in 128 256; do
  AMR_THREADS=$t timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu \
     > gpurun_out/k3_bench_$t.json 2> gpurun_out/k3_bench_$t.err
done
timeout 1200 python -m pytest tests/ -q -m gpu > gpurun_out/k3_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/k3_tests.log
