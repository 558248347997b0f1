# launch list of the backward row per gradient layout (tuning helper)
cd $GRAFT_REPO_ROOT
for lay in v4 planar; do
  VPB_BWD_LAYOUT=$lay ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_backward|k_grad|k_march_rays|Fill|memset" --csv \
    --log-file gpurun_out/bwd_launch_$lay.csv python bench_rows.py --rows backward --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
  VPB_BWD_LAYOUT=$lay python bench_rows.py --rows backward,fit --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | cut -c1-200
done
