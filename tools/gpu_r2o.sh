python -m pytest tests/test_gpu_parity.py tests/test_gpu_domains.py -q -x > gpurun_out/pytest_it.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_it.log
python tools/variants.py time 100 it0 it1 it0 it1 2>&1 | tee gpurun_out/variants9.log
