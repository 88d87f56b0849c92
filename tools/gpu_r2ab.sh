python -m pytest tests/test_gpu_parity.py tests/test_gpu_domains.py -q -x > gpurun_out/pytest_pf.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_pf.log
python tools/variants.py time 100 pf0 pf1 pf0 pf1 2>&1 | tee gpurun_out/variants19.log
