#!/usr/bin/env python
"""Print the key counters, top stalls and instruction mix of an ncu report (here, no GPU).
   python scripts/ncu_quick.py <report.ncu-rep>"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
want = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'smsp__inst_executed.sum',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'launch__registers_per_thread', 'launch__grid_size',
        'launch__block_size', 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'l1tex__throughput.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__cycles_elapsed.avg.per_second',
        'lts__t_sector_hit_rate.pct', 'sm__throughput.avg.pct_of_peak_sustained_elapsed']
for w in want:
    if w in h:
        i = h.index(w)
        print(f'  {w} = {v[i]} {u[i]}')
st = [(float(v[i].replace(',', '')), h[i]) for i in range(len(h))
      if h[i].startswith('smsp__average_warps_issue_stalled') and h[i].endswith('per_issue_active.ratio') and v[i]]
st.sort(reverse=True)
print('  stalls', [(round(a, 2), b.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''))
                   for a, b in st[:9]])
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hh = rows[1]
ie, si, ws = hh.index('Instructions Executed'), hh.index('Source'), hh.index('Warp Stall Sampling (All Samples)')
cnt, stc = collections.Counter(), collections.Counter()
tot = 0
for r in rows[2:]:
    try:
        n = int(r[ie])
    except (ValueError, IndexError):
        continue
    op = r[si].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith('@') else op[0]
    o = o if o.startswith(('LDS', 'STS', 'LDG', 'STG')) else o.split('.')[0]
    cnt[o] += n
    tot += n
    stc[o] += int(r[ws] or 0)
print('  inst total', tot, ' top:', ', '.join(f'{o} {n / tot:.3f}' for o, n in cnt.most_common(14)))
print('  stall samples by opcode:', ', '.join(f'{o} {n}' for o, n in stc.most_common(10)))
