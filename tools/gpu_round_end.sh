# round-end evidence on the GPU box: full GPU suite, smoke, the driver's bench command
# (twice), the default bench, the reference arm, the ncu launch list of the
# driver's window and full captures of k_rows / k_node_warp at step 15 inside it
# (bench.py first warms the process up on an 8x8 grid: init + 5 steps = 6 k_rows
# and 5 node launches, then the 4a init launch; step t of 4a is k_rows launch
# 7 + t and node launch 5 + t)
python -m pytest tests -m gpu -q -x --durations=8 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_driver.log 2>&1; echo "bench rc=$?"
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_driver2.log 2>&1; echo "bench2 rc=$?"
python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench default rc=$?"
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.log 2>&1; echo "bench ref rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_window.csv \
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_w1.log 2>&1; echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_rows -s 21 -c 1 -o gpurun_out/prof_rows_s15 \
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_w2.log 2>&1; echo "ncu2 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_node -s 19 -c 1 -o gpurun_out/prof_node_s15 \
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_w3.log 2>&1; echo "ncu3 rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_smoke.csv \
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ncu_smoke.log 2>&1; echo "ncu smoke rc=$?"
