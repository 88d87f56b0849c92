"""Per-source-line warp-instruction share of k_rows<5> from an ncu report,
for a line range:  python tools/ncu_lines.py REPORT SRC_DIR FIRST LAST"""
import collections
import csv
import re
import subprocess
import sys

rep, sdir, lo, hi = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
subprocess.run(['nvcc', '-gencode', 'arch=compute_100a,code=sm_100a', '-O3', '-lineinfo',
                '-std=c++17', '-cubin', '-o', '/tmp/sec.cubin', f'{sdir}/tsim_rows.cu'],
               check=True, capture_output=True)
dis = subprocess.run(['nvdisasm', '-g', '-c', '/tmp/sec.cubin'], capture_output=True,
                     text=True).stdout.split('\n')
fn = last = None
amap = {}
for ln in dis:
    m = re.search(r'\.text\.(\S+):', ln)
    if m:
        fn = m.group(1)
    m = re.search(r'//## File "(.*)", line (\d+)', ln)
    if m and m.group(1).endswith('tsim_rows.cu'):
        last = int(m.group(2))
    m = re.search(r'/\*([0-9a-f]{4,})\*/', ln)
    if m and fn and 'k_rowsILi5E' in fn:
        amap[int(m.group(1), 16)] = last
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
ie, st, ad = (h.index('Instructions Executed'), h.index('Warp Stall Sampling (All Samples)'),
              h.index('Address'))
base = None
per, stall = collections.Counter(), collections.Counter()
for r in rows[2:]:
    if len(r) <= ie or not r[ad].startswith('0x'):
        continue
    a = int(r[ad], 16)
    if base is None:
        base = a
    line = amap.get(a - base)
    per[line] += int(r[ie] or 0)
    stall[line] += int(r[st] or 0)
tot, stot = sum(per.values()), sum(stall.values())
src = open(f'{sdir}/tsim_rows.cu').read().split('\n')
for line in sorted(k for k in per if k is not None and lo <= k <= hi):
    if per[line] > tot * 0.001 or stall[line] > stot * 0.002:
        print(f'{line:5d} {100*per[line]/tot:5.2f}% {100*stall[line]/stot:5.2f}%  {src[line-1].strip()[:90]}')
