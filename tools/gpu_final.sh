# round-end style GPU pass: parity tests, the default bench line, the ncu
# launch list of a short bench command and one full capture of k_rows
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log
python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/ncu1.log 2>&1; echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_rows -s 60 -c 1 -o gpurun_out/prof_rows \
  python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/ncu2.log 2>&1; echo "ncu2 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_node -s 60 -c 1 -o gpurun_out/prof_node \
  python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/ncu3.log 2>&1; echo "ncu3 rc=$?"
