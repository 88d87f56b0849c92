python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
python tools/variants.py time 100 ppf0 ppf1:960 ppf0:960 ppf1:960 ppf0 2>&1 | tee gpurun_out/variants12.log
