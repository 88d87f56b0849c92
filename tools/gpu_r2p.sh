python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -k "not config5 and not config3 and not config2" > gpurun_out/pytest_it2.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_it2.log
python tools/variants.py time 100 it1 it2 it1 it2 2>&1 | tee gpurun_out/variants10.log
