# cfg3 bench (configs[2], cubic) and the slow bit-exact cfg3-vs-oracle test
cd ${GRAFT_REPO_ROOT:-.}
python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_cfg3.log 2>&1; tail -1 gpurun_out/bench_cfg3.log | cut -c1-1500
AMR_SLOW=1 timeout 1500 python -m pytest tests/test_parity_large_gpu.py -k cfg3 -q -rA > gpurun_out/parity_cfg3.log 2>&1; grep -E "passed|failed|PASSED|FAILED" gpurun_out/parity_cfg3.log | tail -3
