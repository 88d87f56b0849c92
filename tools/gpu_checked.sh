python -m pytest -q -x tests/test_gpu_checked.py > gpurun_out/checked.log 2>&1; echo "checked rc=$?"; tail -30 gpurun_out/checked.log
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_after_checked.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_after_checked.log | cut -c1-300
