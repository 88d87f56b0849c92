python -m pytest tests/test_gpu_domains.py tests/test_gpu_configs.py -q -x -k "local_step or domains or rebalance or load_stat or partition or config5" > gpurun_out/pytest_direct.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_direct.log
python tools/domain_step_times.py 300 > gpurun_out/r2_domain_step_times.json 2> gpurun_out/dst.err; echo "rc=$?"; tail -3 gpurun_out/dst.err
