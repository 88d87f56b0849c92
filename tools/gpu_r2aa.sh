TSIM_LIB=$PWD/build/var_d2/libtsim.so python -m pytest tests/test_gpu_parity.py -q -x -k "bench_flags or config1 or degenerate" > gpurun_out/pytest_d2.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_d2.log
python tools/variants.py time 100 d0 d2 d0 d2 2>&1 | tee gpurun_out/variants18.log
