cd ${GRAFT_REPO_ROOT:-.}
AMR_RS=20 AMR_LIB_PATH=$PWD/build/var/rs20/libamr.so timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -m gpu 2>&1 | tail -2
bash tools/gpu_var.sh base:default: rs20:$PWD/build/var/rs20/libamr.so:AMR_RS=20 base2:default: 2>&1
CFG=cfg3 bash tools/gpu_var.sh rs20_cfg3:$PWD/build/var/rs20/libamr.so:AMR_RS=20 2>&1
