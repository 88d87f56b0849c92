# full parity, the driver's bench line, the ncu evidence of the window, N2 calibration
python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_driver.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_driver.log | cut -c1-400
python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench default rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_window.csv \
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_w1.log 2>&1; echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_rows -s 13 -c 1 -o gpurun_out/prof_rows_w2 \
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_w2.log 2>&1; echo "ncu2 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_node -s 13 -c 1 -o gpurun_out/prof_node_w2 \
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_w3.log 2>&1; echo "ncu3 rc=$?"
python tools/n2_calibrate.py 40 > gpurun_out/r2_perfmodel.md 2> gpurun_out/n2.err; echo "n2 rc=$?"; tail -3 gpurun_out/n2.err
