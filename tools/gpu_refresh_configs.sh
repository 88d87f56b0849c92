# refresh the per-config timings on the final kernels: small configs (launches, graph replay),
# in-process domain step times, config-5 rebalancing, N2 calibration
python tools/small_configs.py 1,2,3,4b > gpurun_out/small.jsonl 2> gpurun_out/small.err; echo "small rc=$?"
python tools/small_configs.py 1,2,3 8 >> gpurun_out/small.jsonl 2>> gpurun_out/small.err; echo "small graph rc=$?"
python tools/domain_step_times.py > gpurun_out/domain_step_times.json 2> gpurun_out/dst.err; echo "dst rc=$?"
python tools/config5_rebalance.py > gpurun_out/config5.json 2> gpurun_out/c5.err; echo "c5 rc=$?"
python tools/n2_calibrate.py 40 > gpurun_out/perfmodel.md 2> gpurun_out/n2.err; echo "n2 rc=$?"; cp profiles/r2_perfmodel.json gpurun_out/ 2>/dev/null
