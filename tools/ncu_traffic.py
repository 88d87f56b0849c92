"""DRAM traffic (and warp instructions) of the dominant kernel from an ncu
--set full report -> profiles/traffic_k_rows.json (read by bench.py for
roofline.traffic and roofline.issue):
  python tools/ncu_traffic.py REPORT [KERNEL_SUBSTR] [NOTE]"""
import csv
import json
import os
import subprocess
import sys

rep = sys.argv[1]
kname = sys.argv[2] if len(sys.argv) > 2 else 'k_rows'
note = sys.argv[3] if len(sys.argv) > 3 else ''
out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units = rows[0], rows[1]


def val(row, key):
    x = float(row[h.index(key)])
    u = units[h.index(key)]
    return x * {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'ns': 1e-9, 'us': 1e-6,
                'usecond': 1e-6, 'msecond': 1e-3, 'nsecond': 1e-9}.get(u, 1)


for r in rows[2:]:
    if kname not in r[h.index('Kernel Name')]:
        continue
    rd, wr = val(r, 'dram__bytes_read.sum'), val(r, 'dram__bytes_write.sum')
    res = {'kernel': r[h.index('Kernel Name')], 'dram_read_bytes': rd, 'dram_write_bytes': wr,
           'traffic_bytes_per_launch': rd + wr,
           'duration_s_under_ncu': val(r, 'gpu__time_duration.sum'),
           'warp_instructions_per_launch': val(r, 'smsp__inst_executed.sum'),
           'issue_active_pct_under_ncu': val(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active'),
           'report': os.path.basename(rep), 'note': note}
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with open(os.path.join(root, 'profiles', 'traffic_k_rows.json'), 'w') as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res))
    break
