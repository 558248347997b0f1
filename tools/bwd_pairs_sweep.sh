# K6b variants and layouts (tuning helper): bash tools/bwd_pairs_sweep.sh lib1 lib2 ...
cd $GRAFT_REPO_ROOT
for lib in "$@"; do
 for lay in ${LAYOUTS:-planar v4}; do
  export VPB_LIB=$(realpath $lib) VPB_BWD_LAYOUT=$lay
  t=$(python -m pytest -q -x -m gpu tests/test_gpu_backward.py -p no:cacheprovider 2>&1 | tail -1)
  r=$(python bench_rows.py --rows backward,fit --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d['row'], d['value'], d.get('ms_per_call', d.get('ms_per_iteration','')), end=' | ')
")
  echo "$(basename $lib) $lay $r $t"
 done
done
