"""Summaries of gpurun_out artefacts (bench lines, ncu launch lists).  Tooling only."""
import csv, json, sys
from collections import defaultdict


def bench(path):
    for l in open(path):
        if l.startswith('{'):
            d = json.loads(l)
            r = d['roofline']
            red = d.get('reduced')
            print(d['config']['workload'][:8], 'value %.0f' % d['value'], 'ms %.2f' % d['ms_per_step'],
                  'far frac %.3f share %.2f avg_ms %.3f' % (r['frac'], r['share_of_step'] or 0, r['avg_launch_ms']),
                  'sweep %.3f' % d['sweep_roofline']['frac'], 'reduced', red and '%.0f' % red['value'],
                  'e2e', d.get('e2e') and '%.0f' % d['e2e']['value'], 'clk', d['clocks'].get('sm_mhz'))


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
    h = rows[hi]
    iid, ik, imn, iv = h.index('ID'), h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value')
    per = defaultdict(dict)
    names = {}
    for r in rows[hi + 1:]:
        if len(r) <= iv or not r[iid].isdigit():
            continue
        per[int(r[iid])][r[imn]] = float(r[iv].replace(',', ''))
        names[int(r[iid])] = r[ik].split('(')[0]
    agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for i, d in per.items():
        a = agg[names[i]]
        t = d.get('gpu__time_duration.sum', 0)
        a[0] += 1
        a[1] += t
        a[2] += d.get('dram__bytes_read.sum', 0) + d.get('dram__bytes_write.sum', 0)
        a[3] += d.get('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 0) * t
    tot = sum(a[1] for a in agg.values())
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:40s} n={a[0]:5d} time={a[1] / 1e6:8.2f} ms share={a[1] / tot:.3f} "
              f"dram/launch={a[2] / a[0] / 1e6:9.1f} MB fp64%={a[3] / max(a[1], 1e-9):.1f}")


if __name__ == '__main__':
    for p in sys.argv[1:]:
        (launches if p.endswith('.csv') else bench)(p)
