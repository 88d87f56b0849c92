#!/bin/bash
for i in 1 2 3 4; do echo "== run $i"; TSIM_TRACE=1 python tools/e2e_breakdown.py 4a 2>&1 | grep "device state\|took\|routes + node\|node outs\|^{"; done
