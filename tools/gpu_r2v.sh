python -m pytest tests/test_gpu_parity.py tests/test_gpu_domains.py -q -x > gpurun_out/pytest_ctab.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_ctab.log
python tools/variants.py time 100 ctab0 ctab ctab0 ctab 2>&1 | tee gpurun_out/variants15.log
