"""Per-source-line / per-section instruction and stall attribution of an
ncu report: python tools/ncu_lines.py REPORT KERNEL_SUBSTR CUBIN_SRC_DIR SRC.cu
(rebuilds the cubin of SRC.cu from CUBIN_SRC_DIR to map SASS addresses to
lines)."""
import collections
import csv
import re
import subprocess
import sys

rep, kname, sdir, src = sys.argv[1:5]
subprocess.run(['nvcc', '-gencode', 'arch=compute_100a,code=sm_100a', '-O3', '-lineinfo',
                '-std=c++17', '-cubin', '-o', f'{sdir}/x.cubin', f'{sdir}/{src}'], check=True,
               capture_output=True)
dis = subprocess.run(['nvdisasm', '-g', '-c', f'{sdir}/x.cubin'], capture_output=True,
                     text=True).stdout.split('\n')
fn = None
cur = None
amap = {}
for ln in dis:
    m = re.search(r'\.text\.(\S+):', ln)
    if m:
        fn = m.group(1)
    m = re.search(r'//## File "(.*)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split('/')[-1], int(m.group(2)))
        continue
    m = re.search(r'/\*([0-9a-f]{4,})\*/', ln)
    if m and fn and kname in fn:
        amap[int(m.group(1), 16)] = cur
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
ie, st, ad = (h.index('Instructions Executed'), h.index('Warp Stall Sampling (All Samples)'),
              h.index('Address'))
te = h.index('Thread Instructions Executed')
base = None
per, stall, thr = collections.Counter(), collections.Counter(), collections.Counter()
for r in rows[2:]:
    if len(r) <= ie or not r[ad].startswith('0x'):
        continue
    a = int(r[ad], 16)
    if base is None:
        base = a
    f = amap.get(a - base, ('?', 0))
    per[f] += int(r[ie] or 0)
    stall[f] += int(r[st] or 0)
    thr[f] += int(r[te] or 0)
tot, stot = sum(per.values()), sum(stall.values())
srcs = {}
print(f'total warp-inst {tot/1e6:.1f}M, stall samples {stot}')
for f, n in sorted(per.items(), key=lambda x: -stall[x[0]] - x[1] / max(tot, 1) * stot)[:45]:
    if f[0] not in srcs:
        try:
            srcs[f[0]] = open(f'{sdir}/{f[0]}').read().split('\n')
        except OSError:
            srcs[f[0]] = []
    line = srcs[f[0]][f[1] - 1].strip()[:64] if f[1] and len(srcs[f[0]]) >= f[1] else ''
    print(f'{f[0][:12]:12s}:{f[1]:4d} inst {100*n/tot:5.1f}% thr {thr[f]/max(n,1):4.1f} '
          f'stall {100*stall[f]/max(stot,1):5.1f}%  {line}')
