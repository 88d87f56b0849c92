# quick GPU check: parity tests then a short bench
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
python bench.py --steps ${STEPS:-300} --warmup 10 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -3 gpurun_out/bench.log
