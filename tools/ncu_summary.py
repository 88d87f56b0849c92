"""Summarise gpurun_out/launches.csv and the ncu reports given on the
command line (raw metrics of every profiled launch)."""
import csv
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__thread_inst_executed_per_inst_executed.ratio', 'launch__registers_per_thread',
        'smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']


def launches(path='gpurun_out/launches.csv'):
    rows = list(csv.reader(open(path)))
    hdr = None
    for r in rows:
        if r and r[0] == 'ID':
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            print(f"{r[hdr.index('Kernel Name')][:44]:44s} {r[hdr.index('Grid Size')]:>14s} "
                  f"{r[hdr.index('Metric Value')]:>10s} ns")


def raw(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h = r[0]
    for row in r[2:]:
        name = row[h.index('Kernel Name')][:30]
        vals = {k.split('__')[1].split('.')[0]: row[h.index(k)] for k in KEYS if k in h}
        print(rep, name, vals)


if __name__ == '__main__':
    launches()
    for rep in sys.argv[1:]:
        raw(rep)
