python -m pytest tests/test_gpu_domains.py -q -x -k "local_step or rebalance or load_stat" > gpurun_out/pytest_local.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_local.log
python tools/variants.py time 100 z0 zskip zm3 zm3s z0 zskip 2>&1 | tee gpurun_out/variants6.log
