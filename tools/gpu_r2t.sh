TSIM_LIB=$PWD/build/var_rkr/libtsim.so python -m pytest tests/test_gpu_parity.py -q -x -k "bench_flags or config1 or dense" > gpurun_out/pytest_rkr.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_rkr.log
python tools/variants.py time 100 ppf0 rkr ppf0 rkr 2>&1 | tee gpurun_out/variants13.log
