# Ray-batch kernel sweep (tuning helper): per variant, the backward/train parity tests and the
# backward + fit rows. Usage: bash tools/sweep_rays.sh build/variants/libvpb_*.so
for lib in "$@"; do
  export VPB_LIB=$(realpath $lib)
  t=$(python -m pytest -q -x -m gpu tests/test_gpu_backward.py tests/test_gpu_train.py 2>&1 | tail -1)
  r=$(python bench_rows.py --rows backward,fit --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d['row'], d['value'], d.get('ms_per_call', d.get('ms_per_iteration','')), end=' | ')
")
  echo "$(basename $lib) $r $t"
done
