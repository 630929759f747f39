cd ${GRAFT_REPO_ROOT:-.}
timeout 2400 python -m pytest tests -q -x -m gpu 2>&1 | tail -8 > gpurun_out/exp15_all.txt
cat gpurun_out/exp15_all.txt
for i in 1 2 3; do
  python bench.py --no-cpu --side none --steps 10 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('pipelined LTS %.2f G e2e %.2f G (%.3f) eng %.2f s mesh %.2f s' % (d['value']/1e9, d['e2e']['value']/1e9, d['e2e']['value']/d['value'], d['engine_build_s'], d['mesh_build_s']))"
done
python bench.py --no-cpu --side none --steps 10 --warmup 3 --e2e-serial 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('serial    LTS %.2f G e2e %.2f G (%.3f)' % (d['value']/1e9, d['e2e']['value']/1e9, d['e2e']['value']/d['value']))"
