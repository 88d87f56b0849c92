# ncu of the row and node kernels on config 4a at steady state (WARM warm-up
# steps); every ncu run is chained after a clean plain run of the same command
W=${WARM:-300}
python tools/prof.py $W > gpurun_out/prof_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -s $((2*W)) -c 12 --csv --log-file gpurun_out/launches.csv python tools/prof.py $W > gpurun_out/ncu1.log 2>&1
echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_rows -s $((W+3)) -c 1 -o gpurun_out/prof_rows python tools/prof.py $W > gpurun_out/ncu2.log 2>&1
echo "ncu2 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_node -s $((W)) -c 1 -o gpurun_out/prof_node python tools/prof.py $W > gpurun_out/ncu3.log 2>&1
echo "ncu3 rc=$?"
