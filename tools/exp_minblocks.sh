cd $GRAFT_REPO_ROOT
bash tests/gpu_parity.sh > gpurun_out/parity9.log 2>&1; grep -E "passed|failed" gpurun_out/parity9.log | tail -3
python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench9_mb3.log 2>&1; tail -1 gpurun_out/bench9_mb3.log | cut -c1-200; grep -o '"gts": {[^}]*}' gpurun_out/bench9_mb3.log
AMR_NVCC_FLAGS="-DAMR_MIN_BLOCKS=2" python paper_2011_10570_b200/build.py --force > /dev/null 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench9_mb2.log 2>&1; tail -1 gpurun_out/bench9_mb2.log | cut -c1-200; grep -o '"gts": {[^}]*}' gpurun_out/bench9_mb2.log
AMR_NVCC_FLAGS="-DAMR_MIN_BLOCKS=4" python paper_2011_10570_b200/build.py --force > /dev/null 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench9_mb4.log 2>&1; tail -1 gpurun_out/bench9_mb4.log | cut -c1-200; grep -o '"gts": {[^}]*}' gpurun_out/bench9_mb4.log
