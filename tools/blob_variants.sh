# Compile-time variants of the blob kernel (AMR_NVCC_FLAGS), cfg2 bench each, then the product build.
# usage: VARIANTS="none -DAMR_BLOB_MIN_BLOCKS=3" bash tools/blob_variants.sh   ("none" = product flags)
cd ${GRAFT_REPO_ROOT:-.}
for fl in ${VARIANTS:-none}; do
  f="$fl"; [ "$fl" = none ] && f=""
  AMR_NVCC_FLAGS="$f" python -m paper_2011_10570_b200.build --force > /dev/null
  python bench.py --steps 5 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$fl] LTS', round(d['value']/1e9,2), 'GTS', round(d['gts']['value']/1e9,2), 'frac', round(d['roofline']['frac'],3))"
done
python -m paper_2011_10570_b200.build --force > /dev/null
