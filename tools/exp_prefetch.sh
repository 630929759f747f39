cd ${GRAFT_REPO_ROOT:-.}
bash tests/gpu_parity.sh > gpurun_out/parity_pf.log 2>&1; grep -E "passed|failed" gpurun_out/parity_pf.log | tail -2
for pf in 1 0; do
  AMR_PREFETCH=$pf python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_pf$pf.log 2>&1
  echo "prefetch=$pf"; tail -1 gpurun_out/bench_pf$pf.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['gts']['value'], d['roofline']['frac'], d['e2e']['value'])"
done
