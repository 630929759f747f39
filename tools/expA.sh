cd ${GRAFT_REPO_ROOT:-.}
bash tools/gpu_var.sh base:default: prek:$PWD/build/var/prek/libamr.so: base2:default: prek2:$PWD/build/var/prek/libamr.so: 2>&1
