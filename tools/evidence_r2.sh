# copy the round-end evidence (tools/gpu_round_end.sh output in gpurun_out/) into
# profiles/: bench lines, launch lists, raw ncu pages, traffic, the summary
set -e
tail -1 gpurun_out/bench_driver.log > profiles/r2_bench_driver_window.json
tail -1 gpurun_out/bench_driver2.log > profiles/r2_bench_driver_window_repeat.json
tail -1 gpurun_out/bench_default.log > profiles/r2_bench_default.json
tail -1 gpurun_out/bench_ref.log > profiles/r2_bench_reference.json
cp gpurun_out/launches_window.csv profiles/r2_launches_window.csv
cp gpurun_out/launches_smoke.csv profiles/r2_launches_smoke.csv
ncu -i gpurun_out/prof_rows_s15.ncu-rep --page raw --csv > profiles/r2_ncu_full_window_k_rows.csv
ncu -i gpurun_out/prof_node_s15.ncu-rep --page raw --csv > profiles/r2_ncu_full_window_k_node_warp.csv
python tools/ncu_traffic.py gpurun_out/prof_rows_s15.ncu-rep k_rows "driver window (bench.py --steps 20 --warmup 5), k_rows launch of step 15, round-2 final kernels ($(git rev-parse --short HEAD))"
