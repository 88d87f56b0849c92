#!/bin/bash
python -m pytest tests/test_gpu_inputs.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_di.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_di.log
for i in 1 2 3; do for m in packed checked; do if [ $m = checked ]; then export TSIM_LOAD_CHECKED=1; else unset TSIM_LOAD_CHECKED; fi
echo "$m $(TSIM_TRACE=1 python tools/e2e_breakdown.py 4a 2>&1 | grep 'out-slots')"; done; done
