python -m pytest tests/test_gpu_parity.py -q -x -k "bench_flags or config1 or history or graph_replay_grid" > gpurun_out/pytest_wf.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_wf.log
python tools/variants.py time 100 wf0 wf1 wf0 wf1 2>&1 | tee gpurun_out/variants17.log
