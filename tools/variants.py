"""Tuning variants of libtsim: build (here) and time (on the GPU box).

  python tools/variants.py build NAME:-DFLAG=1,-DX=2 ...   -> build/var_NAME/libtsim.so
  python tools/variants.py time STEPS NAME[:group_cells] ... -> one JSON line per variant
Each timing runs config 4a in a fresh process with TSIM_LIB pointing at the
variant; 'base' is the in-tree library.  Reported: the driver's bench window
(steps 6..25: warm-up 5, 20 timed) and a steady-state window after 225
steps, ms per step and per k_rows launch.

  python tools/variants.py build_git REV NAME   -> build/var_NAME from the sources at REV"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def build(specs):
    from paper_cs_0105004_b200 import build as b
    for spec in specs:
        name, _, flags = spec.partition(':')
        out = os.path.join(ROOT, 'build', f'var_{name}')
        os.makedirs(out, exist_ok=True)
        cmd = (['/usr/local/cuda/bin/nvcc'] + b.NVCC_FLAGS + [f for f in flags.split(',') if f] +
               [os.path.join(b.HERE, s) for s in b.SRCS] + ['-o', os.path.join(out, 'libtsim.so')])
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise SystemExit(r.stderr)
        regs = [ln for ln in r.stderr.split('\n') if 'registers' in ln]
        print(name, flags, regs[-1].strip() if regs else '')


CHILD = r'''
import json, sys
sys.path.insert(0, {root!r})
import scenarios
import paper_cs_0105004_b200 as tsim
scn = scenarios.config('4a')
sim = tsim.Sim(p_slow=scn.p_slow, seed=scn.seed, flags=tsim.FLAG_FUSED, group_cells={gc})
sim.load(scn)
sim.init(0)
sim.step(5)           # the driver's window: --warmup 5 --steps 20
sim.step(20)
w = sim.last_timing()
sim.step(200)         # steady state
sim.step({steps})
tm = sim.last_timing()
print(json.dumps(dict(win_ms_step=w['total_ms'] / 20, win_ms_move=w['move_ms'] / max(1, w['move_launches']),
                      ms_step=tm['total_ms'] / {steps}, ms_move=tm['move_ms'] / max(1, tm['move_launches']))))
'''


def time(steps, specs):
    for spec in specs:
        name, _, gc = spec.partition(':')
        env = dict(os.environ)
        if name.endswith('+nopdl'):
            name = name[:-len('+nopdl')]
            env['TSIM_NO_PDL'] = '1'
        if name != 'base':
            env['TSIM_LIB'] = os.path.join(ROOT, 'build', f'var_{name}', 'libtsim.so')
        code = CHILD.format(root=ROOT, gc=int(gc or 0), steps=steps)
        r = subprocess.run([sys.executable, '-c', code], env=env, capture_output=True, text=True,
                           timeout=900)
        line = r.stdout.strip().split('\n')[-1] if r.returncode == 0 else r.stderr[-300:]
        print(json.dumps({'variant': spec, 'result': line}), flush=True)


def build_git(rev, name):
    """the kernel sources of an older commit (A/B timing against it)"""
    import shutil
    import tempfile
    from paper_cs_0105004_b200 import build as b
    tmp = tempfile.mkdtemp()
    subprocess.run(f"git -C {ROOT} archive {rev} paper_cs_0105004_b200/csrc include | tar -x -C {tmp}",
                   shell=True, check=True)
    out = os.path.join(ROOT, 'build', f'var_{name}')
    os.makedirs(out, exist_ok=True)
    srcs = [os.path.join(tmp, 'paper_cs_0105004_b200', s) for s in b.SRCS]
    r = subprocess.run(['/usr/local/cuda/bin/nvcc'] + b.NVCC_FLAGS + srcs +
                       ['-o', os.path.join(out, 'libtsim.so')], capture_output=True, text=True)
    shutil.rmtree(tmp)
    if r.returncode:
        raise SystemExit(r.stderr)
    print(name, rev, 'built')


if __name__ == '__main__':
    if sys.argv[1] == 'build_git':
        build_git(sys.argv[2], sys.argv[3])
    elif sys.argv[1] == 'build':
        build(sys.argv[2:])
    else:
        time(int(sys.argv[2]), sys.argv[3:])
