python -m pytest tests/test_gpu_parity.py tests/test_gpu_domains.py -q -x > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_quick.log
python tools/variants.py time 100 r1 c1 v2a v2b v2b_nosp v2b_nork v2b_nospnork v2b_m5:992 v2b_m6:768 v2b_m5nork:992 r1 v2b 2>&1 | tee gpurun_out/variants2.log
