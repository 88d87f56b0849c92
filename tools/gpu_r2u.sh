python -m pytest tests/test_gpu_parity.py tests/test_gpu_domains.py tests/test_gpu_validation.py -q -x > gpurun_out/pytest_nk.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_nk.log
python tools/variants.py time 100 nk0 nk nk0 nk 2>&1 | tee gpurun_out/variants14.log
