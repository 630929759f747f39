cd ${GRAFT_REPO_ROOT:-.}
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_ranks_gpu.py tests/test_parity_large_gpu.py -q -x -m gpu 2>&1 | tail -3
bash tools/gpu_var.sh new:default: base:$PWD/build/var/base/libamr.so: new2:default: 2>&1
CFG=cfg3 bash tools/gpu_var.sh new_cfg3:default: base_cfg3:$PWD/build/var/base/libamr.so: 2>&1
