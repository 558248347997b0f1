# backward row over library variants (tuning helper): bash tools/variant_backward.sh lib...
cd $GRAFT_REPO_ROOT
for lib in "$@"; do
  r=$(VPB_LIB=$(realpath $lib) python bench_rows.py --rows backward --steps 30 --warmup 3 --no-cpu-baseline 2>/dev/null | grep -o '"value": [0-9.]*')
  echo "$(basename $lib) $r"
done
