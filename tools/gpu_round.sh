set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q > gpurun_out/r1_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r1_pytest_gpu.log
python bench.py --steps 300 --warmup 10 > gpurun_out/r1_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r1_bench.log
python tools/prof.py > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python tools/prof.py > gpurun_out/ncu1.log 2>&1
echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_rows -s 4 -c 2 -o gpurun_out/prof_rows python tools/prof.py > gpurun_out/ncu2.log 2>&1
echo "ncu2 rc=$?"
