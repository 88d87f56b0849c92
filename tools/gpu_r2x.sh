TSIM_LIB=$PWD/build/var_ra1/libtsim.so python -m pytest tests/test_gpu_parity.py -q -x -k "bench_flags or config1 or degenerate" > gpurun_out/pytest_ra1.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_ra1.log
python tools/variants.py time 100 ra0 ra1 ra0 ra1 2>&1 | tee gpurun_out/variants16.log
