# One GPU iteration: parity (-x), phase probe, bench (cfg2, no CPU leg).
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-it}
bash tests/gpu_parity.sh -x > gpurun_out/parity_$TAG.log 2>&1; grep -E "passed|failed" gpurun_out/parity_$TAG.log | tail -2
python tools/phase_probe.py > gpurun_out/phase_$TAG.txt 2>&1; python tools/phase_probe.py --mode lts >> gpurun_out/phase_$TAG.txt 2>&1; cat gpurun_out/phase_$TAG.txt
python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_$TAG.log 2>&1
tail -1 gpurun_out/bench_$TAG.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('LTS', d['value'], 'GTS', d['gts']['value'], 'frac', d['roofline']['frac'], 'e2e', d['e2e']['value'])"
