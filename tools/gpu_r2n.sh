TSIM_LIB=$PWD/build/var_da1/libtsim.so python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_da1.log 2>&1; echo "pytest da1 rc=$?"; tail -2 gpurun_out/pytest_da1.log
python tools/variants.py time 100 da0 da700 da800 da1 da0 da700 2>&1 | tee gpurun_out/variants8.log
