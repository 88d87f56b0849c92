#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_gpu_inputs.py tests/test_gpu_api.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_di.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_di.log
for i in 1 2 3; do
for g in dyn static; do echo "== $g"; if [ $g = static ]; then export TSIM_STATIC_CHUNKS=1; else unset TSIM_STATIC_CHUNKS; fi
TSIM_TRACE=1 python tools/e2e_breakdown.py 4a 2>&1 | grep -v "^\[tsim init\] *$"; done; done
