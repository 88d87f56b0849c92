#!/bin/bash
for i in 1 2 3 4 5 6; do echo "== run $i"; TSIM_TRACE=1 python tools/e2e_breakdown.py 4a 2>&1 | grep "tsim init\|^{"; done
