# Ray-batch kernels A/B (tuning helper): parity tests + backward/fit rows per library variant.
# Usage: bash tools/rays_sweep.sh build/variants/libvpb_*.so
for lib in "$@"; do
  export VPB_LIB=$(realpath $lib)
  t=$(python -m pytest -q -x -m gpu tests/test_gpu_backward.py tests/test_gpu_train.py tests/test_gpu_parity.py -k "march or backward or train or adam or eval or bvh or ray" -p no:cacheprovider 2>&1 | tail -1)
  r=$(python bench_rows.py --rows backward,fit --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d['row'], d['value'], d.get('ms_per_call', d.get('ms_per_iteration','')), end=' | ')
")
  echo "$(basename $lib) $r $t"
done
