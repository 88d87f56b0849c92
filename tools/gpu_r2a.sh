# round 2: host probe, GPU tests with durations, the driver's bench command
free -g > gpurun_out/host.txt; nproc >> gpurun_out/host.txt; nvidia-smi --query-gpu=name,memory.total --format=csv >> gpurun_out/host.txt
python -m pytest tests -m gpu -q --durations=30 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -45 gpurun_out/pytest_gpu.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_driver.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_driver.log | cut -c1-600
