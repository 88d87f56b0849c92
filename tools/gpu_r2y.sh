TSIM_TRACE=1 python tools/e2e_breakdown.py 4a > gpurun_out/e2e_breakdown.txt 2>&1; echo "e2e rc=$?"; tail -12 gpurun_out/e2e_breakdown.txt
