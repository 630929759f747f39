#!/bin/bash
# What the driver runs at round end, in one call: GPU tests, smoke(), both bench arms.
cd ${GRAFT_REPO_ROOT:-.}
[ -n "$SKIP_TESTS" ] || timeout 2400 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; tail -c 300 gpurun_out/final_ref.json
SECONDS=0; timeout 1500 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench wall ${SECONDS}s"
python - <<'PY'
import json
d=json.loads(open("gpurun_out/final_bench.json").read().strip().splitlines()[-1])
print("LTS %.2f G GTS %.2f G e2e %.2f G frac %.3f launches %d" % (d["value"]/1e9, d["gts"]["value"]/1e9, d["e2e"]["value"]/1e9, d["roofline"]["frac"], d["gpu_launches"]))
print({k: round(v["value"]/1e9, 2) for k, v in d["other_configs"].items()}, d["clocks"])
PY
