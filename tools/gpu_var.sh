# GPU parity tests (TESTS, default: the parity files), then timings of the tuning variants given in $VARS
python -m pytest ${TESTS:-tests/test_gpu_parity.py tests/test_gpu_configs.py} -x -q > gpurun_out/pytest_var.log 2>&1; rc=$?; echo "pytest rc=$rc"; tail -2 gpurun_out/pytest_var.log
python tools/variants.py time ${STEPS:-200} $VARS 2>&1 | tee gpurun_out/variants.log
