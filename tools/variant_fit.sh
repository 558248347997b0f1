# fit split over library variants (tuning helper): bash tools/variant_fit.sh lib...
cd $GRAFT_REPO_ROOT
for lib in "$@"; do
  for rep in 1 2; do
    echo "$(basename $lib) $(VPB_LIB=$(realpath $lib) python tools/fit_breakdown.py 2>&1 | tail -1)"
  done
done
