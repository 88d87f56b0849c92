python tools/domain_step_times.py 300 > gpurun_out/r2_domain_step_times.json 2> gpurun_out/dst.err; echo "rc=$?"; tail -3 gpurun_out/dst.err
