python tools/variants.py time 100 y0:1344 ya1:1344 ya2:1344 yav:1344 yal:1344 yaall:1344 y0:1344 2>&1 | tee gpurun_out/variants5.log
