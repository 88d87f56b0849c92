#!/bin/bash
python -m pytest tests/test_gpu_api.py tests/test_gpu_parity.py tests/test_gpu_domains.py tests/test_gpu_inputs.py -q -x > gpurun_out/pytest_di.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_di.log
for i in 1 2 3; do python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d[\"value\"]/1e10,3), d[\"e2e\"][\"wall_s\"], d[\"e2e\"][\"phases_s\"])"; done
