#!/bin/bash
# compute-sanitizer memcheck and racecheck over the stage, interface, ghost,
# octree and wavelet kernels (tools/sanitize_run.py); logs in gpurun_out/.
cd ${GRAFT_REPO_ROOT:-.}
python tools/sanitize_run.py > gpurun_out/sanitize_plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/sanitize_plain.log; exit 1; }
for tool in memcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|^ok" gpurun_out/sanitize_$tool.log | tail -3
done
