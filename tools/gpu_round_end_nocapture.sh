# round-end evidence without the ncu full captures (kernels unchanged since
# the last capture): full GPU suite, smoke, the driver's bench command
# (twice), the default bench, the reference arm, the smoke launch list
python -m pytest tests -m gpu -q -x --durations=8 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_driver.log 2>&1; echo "bench rc=$?"
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_driver2.log 2>&1; echo "bench2 rc=$?"
python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench default rc=$?"
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.log 2>&1; echo "bench ref rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_smoke.csv \
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ncu_smoke.log 2>&1; echo "ncu smoke rc=$?"
