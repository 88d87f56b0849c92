python tools/variants.py time 100 r1 v2b_nosp x0 x0:1344 xitab xd2 xfs xcs xall r1 x0 xall 2>&1 | tee gpurun_out/variants4.log
