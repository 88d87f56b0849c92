python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_it3.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_it3.log
python tools/variants.py time 100 it2 it3 it2 it3 2>&1 | tee gpurun_out/variants11.log
