set -x
timeout 500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/smoke.log
timeout 300 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 200 python bench.py --tile-shard > gpurun_out/bench_shard.json 2> gpurun_out/bench_shard.err
timeout 600 python bench_rows.py > gpurun_out/rows.jsonl 2> gpurun_out/rows.err
timeout 300 python tools/sweep.py paper_2103_01954_b200/libvpb.so > gpurun_out/sweep_final.txt 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --quick --steps 2 --warmup 1 > gpurun_out/launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_march_tiles -s 35 -c 1 -o gpurun_out/march_full python bench.py --quick --steps 1 --warmup 3 > gpurun_out/march_full.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bw_launches.csv python bench_rows.py --rows backward --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bw_launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_backward_rays_warp -s 1 -c 1 -o gpurun_out/bw_full python bench_rows.py --rows backward --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bw_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_march_rays_warp -s 1 -c 1 -o gpurun_out/fw_full python bench_rows.py --rows backward --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/fw_full.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fit_launches.csv python bench_rows.py --rows fit --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/fit_launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_adam_update4 -s 1 -c 1 -o gpurun_out/adam_full python bench_rows.py --rows fit --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/adam_full.log 2>&1
