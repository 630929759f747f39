#!/bin/bash
# Bench variants of the stage kernel on one box: each argument is
# "tag:lib_path_or_default:ENV=VAL,ENV=VAL"; prints one summary line per variant.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
CFG=${CFG:-cfg2}
for spec in "$@"; do
  IFS=: read -r tag lib envs <<< "$spec"
  ( [ "$lib" != "default" ] && export AMR_LIB_PATH=$lib
    IFS=, ; for kv in $envs; do [ -n "$kv" ] && export "$kv"; done
    timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --config $CFG > gpurun_out/var_$tag.json 2> gpurun_out/var_$tag.err )
  python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
try:
    d = [json.loads(l) for l in open(f"gpurun_out/var_{tag}.json") if l.startswith("{")][-1]
    print(f"{tag:12s} LTS {d['value']/1e9:6.2f} G  GTS {d['gts']['value']/1e9:6.2f} G  frac {d['roofline']['frac']:.3f}/{d['roofline']['gts_frac']:.3f}  e2e {d['e2e']['value']/1e9:6.2f} G  ms {d['ms_per_step']:.3f}  speedup {d['lts_vs_gts_wall_speedup']:.2f}")
except Exception as e:
    print(tag, "FAILED", e, open(f"gpurun_out/var_{tag}.err").read()[-600:])
PY
done
