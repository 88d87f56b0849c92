# ncu of k_rows inside the driver's window (bench.py --steps 20 --warmup 5):
# launch list, and one full capture of the launch of step ~12
python tools/window_stats.py 4a 40 > gpurun_out/window_stats.txt 2>&1; echo "stats rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_window.csv \
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_w1.log 2>&1; echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_rows -s ${SKIP:-13} -c 1 -o gpurun_out/prof_rows_w \
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_w2.log 2>&1; echo "ncu2 rc=$?"
