python -m pytest tests/test_gpu_parity.py tests/test_gpu_inputs.py tests/test_gpu_api.py -q -x > gpurun_out/pytest_rd.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_rd.log
python tools/e2e_breakdown.py 4a > gpurun_out/e2e_breakdown2.txt 2>&1; echo "e2e rc=$?"; tail -1 gpurun_out/e2e_breakdown2.txt
