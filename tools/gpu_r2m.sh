python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_np.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_np.log
python tools/variants.py time 100 np0 np1 np0 np1 2>&1 | tee gpurun_out/variants7.log
