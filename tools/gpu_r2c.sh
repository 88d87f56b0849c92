# parity of the current kernels, then A/B timing against round 1 (driver window + steady state)
python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_gpu.log
python tools/variants.py time 100 base r1 base r1 2>&1 | tee gpurun_out/variants.log
