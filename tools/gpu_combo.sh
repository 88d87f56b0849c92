python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
[ "$(grep -c failed gpurun_out/pytest_gpu.log)" = "0" ] && bash tools/gpu_prof.sh
