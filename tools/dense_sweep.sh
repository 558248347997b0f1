# dense-tier configuration variants at 32768x8^3 (tuning helper): bash tools/dense_sweep.sh lib...
cd $GRAFT_REPO_ROOT
for lib in "$@"; do
  VPB_LIB=$(realpath $lib) timeout 300 python bench.py --quick --steps 10 --warmup 3 --k 32768 --m 8 --no-sweep \
    --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$(basename $lib)', d['value'], d['roofline']['frac'])"
done
