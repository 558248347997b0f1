cd $GRAFT_REPO_ROOT
for lib in build/variants/libvpb_mb3.so build/variants/libvpb_mb4.so build/variants/libvpb_mb5.so; do
 for lay in v4 planar; do
  export VPB_LIB=$(realpath $lib) VPB_BWD_LAYOUT=$lay
  t=$(python -m pytest -q -x -m gpu tests/test_gpu_backward.py tests/test_gpu_train.py -p no:cacheprovider 2>&1 | tail -1)
  r=$(python bench_rows.py --rows backward,fit --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d['row'], d['value'], d.get('ms_per_call', d.get('ms_per_iteration','')), end=' | ')
")
  echo "$(basename $lib) $lay $r $t"
 done
done
