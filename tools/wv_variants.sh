# Wavelet-kernel variants on the GPU box: recompile amr_wavelet.cu with
# -D flags, link against the in-tree objects, bench each (no CPU leg).
cd ${GRAFT_REPO_ROOT:-.}
NV=/usr/local/cuda/bin/nvcc
# VARIANTS: space-separated, flags inside one variant joined by ","
for V0 in ${VARIANTS:-"-DWV_MINB=2,-DWV_INTMAX=1 -DWV_MINB=3,-DWV_INTMAX=0"}; do
  V=$(echo "$V0" | tr ',' ' ')
  tag=$(echo "$V0" | tr -d ',=-')
  $NV -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC $V -c paper_2011_10570_b200/csrc/amr_wavelet.cu -o /tmp/wv_$tag.o || continue
  $NV -gencode arch=compute_100a,code=sm_100a -shared -o /tmp/libv_$tag.so /tmp/wv_$tag.o paper_2011_10570_b200/_lib/amr_kernels.o paper_2011_10570_b200/_lib/amr_mesh.o -lgomp || continue
  echo "== $V"
  AMR_LIB_PATH=/tmp/libv_$tag.so python tools/bench_wavelet.py --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms', round(d['ms_per_launch'],4), 'frac', round(d['roofline']['frac'],3))"
  AMR_LIB_PATH=/tmp/libv_$tag.so python -m pytest tests/test_wavelet_gpu.py -q -x -k "bit_exact or random_values" 2>&1 | tail -1
done
