# run the GPU parity suite on a gpurun box; full log in gpurun_out/parity.log
cd ${GRAFT_REPO_ROOT:-.}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -q -rA "$@" 2>&1
