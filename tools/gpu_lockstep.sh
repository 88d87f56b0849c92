python -m pytest tests -m gpu -x -q -k "not validation" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for ls in 0 8 16 20; do echo "lockstep=$ls"; TS_ROWS_LOCKSTEP=$ls python tools/sweep.py 1024; done
TS_ROWS_LOCKSTEP=16 python -m pytest tests/test_gpu_parity.py -x -q -k "config1_full or big_grid or portland" 2>&1 | tail -2
