# GPU parity tests, then timings of the tuning variants given in $VARS
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; rc=$?; echo "pytest rc=$rc"; tail -3 gpurun_out/pytest_gpu.log
python tools/variants.py time ${STEPS:-200} $VARS 2>&1 | tee gpurun_out/variants.log
