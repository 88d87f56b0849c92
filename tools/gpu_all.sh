# GPU tests; if green: short bench and steady-state profiles
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; rc=$?; echo "pytest rc=$rc"; tail -4 gpurun_out/pytest_gpu.log
[ $rc = 0 ] || exit 1
python bench.py --steps ${STEPS:-300} --warmup 10 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log
[ "${PROF:-1}" = 1 ] && bash tools/gpu_prof.sh
