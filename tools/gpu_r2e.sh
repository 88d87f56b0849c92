python -m pytest tests/test_gpu_parity.py tests/test_gpu_domains.py tests/test_gpu_native.py -q -x > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_quick.log
python tools/variants.py time 100 r1 v2b_nosp v3 v3_d1 v3:1088 r1 v3 2>&1 | tee gpurun_out/variants3.log
