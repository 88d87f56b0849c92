"""Dynamic (ncu-measured) warp-instruction and stall share of k_rows per
source section (// ---- markers), attributing inlined helper lines to the
last tsim_rows.cu line seen:  python tools/ncu_sections.py REPORT SRC_DIR"""
import collections
import csv
import re
import subprocess
import sys

rep, sdir = sys.argv[1:3]
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
src = open(f'{sdir}/tsim_rows.cu').read().split('\n')
k0 = next(i for i, l in enumerate(src) if 'k_rows(const StepParams' in l) + 1
secs = [(k0, 'kernel setup')] + [(i + 1, l.strip()[:60]) for i, l in enumerate(src)
                                 if '// ----' in l and i + 1 > k0]
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
    name = 'helpers (before kernel)'
    if line is not None and line >= k0:
        for s, t in secs:
            if s <= line:
                name = f'{s:4d} {t}'
    per[name] += int(r[ie] or 0)
    stall[name] += int(r[st] or 0)
tot, stot = sum(per.values()), sum(stall.values())
print(f'total warp-inst {tot/1e6:.1f}M  stall samples {stot}')
for k in sorted(per):
    print(f'{100*per[k]/tot:5.1f}% inst  {100*stall[k]/max(stot,1):5.1f}% stall  {k}')
