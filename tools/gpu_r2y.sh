#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2 3; do
for st in reg staged; do echo "route $st"; if [ $st = staged ]; then export TSIM_ROUTE_STAGED=1; else unset TSIM_ROUTE_STAGED; fi; TSIM_TRACE=1 python tools/e2e_breakdown.py 4a 2>&1 | grep -v "^\[tsim init\] *$" | grep "records\|general\|out-slots\|took\|tiles\|pending\|generate\|node outs\|routes +"; done
done
