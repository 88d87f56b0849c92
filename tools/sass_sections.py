"""Static SASS instruction count of k_rows per source section (// ---- markers)."""
import collections
import re
import subprocess
import sys

src_dir = sys.argv[1] if len(sys.argv) > 1 else 'paper_cs_0105004_b200/csrc'
subprocess.run(['nvcc', '-gencode', 'arch=compute_100a,code=sm_100a', '-O3', '-lineinfo',
                '-std=c++17', '-cubin', '-o', '/tmp/sec.cubin', f'{src_dir}/tsim_rows.cu'],
               check=True, capture_output=True)
dis = subprocess.run(['nvdisasm', '-g', '-c', '/tmp/sec.cubin'], capture_output=True,
                     text=True).stdout.split('\n')
fn = cur = last = None
cnt = collections.Counter()
for ln in dis:
    m = re.search(r'\.text\.(\S+):', ln)
    if m:
        fn = m.group(1)
    m = re.search(r'//## File "(.*)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split('/')[-1], int(m.group(2)))
        if cur[0] == 'tsim_rows.cu':
            last = cur[1]
    if re.search(r'/\*[0-9a-f]{4,}\*/', ln) and fn and 'k_rowsILi5E' in fn:
        cnt[last] += 1
src = open(f'{src_dir}/tsim_rows.cu').read().split('\n')
k0 = next(i for i, l in enumerate(src) if 'k_rows(const StepParams' in l) + 1
secs = [(k0, 'kernel setup')] + [(i + 1, l.strip()[:64]) for i, l in enumerate(src)
                                 if '// ----' in l and i + 1 > k0]
agg = collections.Counter()
for line, n in cnt.items():
    name = 'helpers (before kernel)'
    if line is not None and line >= k0:
        for a, t in secs:
            if a <= line:
                name = f'{a:4d} {t}'
    agg[name] += n
print('total', sum(cnt.values()))
for k, v in sorted(agg.items()):
    print(f'{v:6d}  {k}')
