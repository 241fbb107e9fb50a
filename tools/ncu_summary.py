"""Text summary of ncu captures for profiles/ (experiment tooling):
key metrics + top stall reasons per captured kernel, and the per-kernel
totals of a launch-list CSV.
  python tools/ncu_summary.py launches.csv|- rep1.ncu-rep [rep2.ncu-rep ...]"""
import csv, io, subprocess, sys
from collections import defaultdict

METRICS = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
           "launch__grid_size", "launch__registers_per_thread",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active"]
STALLS = ["wait", "selected", "math_pipe_throttle", "not_selected", "long_scoreboard",
          "short_scoreboard", "dispatch_stall", "branch_resolving", "mio_throttle", "barrier",
          "no_instruction", "lg_throttle", "sleeping"]

def rep_summary(rep):
    q = METRICS + [f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio" for s in STALLS]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(q)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    lines = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        lines.append(f"===== {d['Kernel Name'][:70]}")
        for mname in METRICS:
            if mname in d:
                lines.append(f"  {mname:<70} {d[mname]}")
        st = []
        for s in STALLS:
            k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if k in d and d[k]:
                try:
                    st.append((float(d[k]), s))
                except ValueError:
                    pass
        st.sort(reverse=True)
        lines.append("  stalls/issue: " + ", ".join(f"{s} {v:.2f}" for v, s in st if v >= 0.03))
    return lines

def launch_summary(path):
    rows = list(csv.reader(open(path)))
    i0 = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[i0]
    iid, ik, imn, iv = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    dur = {}
    name = {}
    for r in rows[i0 + 1:]:
        if len(r) > iv and r[iid].isdigit() and r[imn] == "gpu__time_duration.sum":
            dur[int(r[iid])] = float(r[iv].replace(",", ""))
            name[int(r[iid])] = r[ik].split("(")[0]
    agg = defaultdict(lambda: [0, 0.0])
    for i, t in dur.items():
        agg[name[i]][0] += 1
        agg[name[i]][1] += t
    tot = sum(v[1] for v in agg.values())
    lines = ["# launch list of one bench step (ncu --metrics gpu__time_duration.sum, cold/serialised):"]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"#  {n:5d} launches {t / 1e6:9.3f} ms {100 * t / tot:5.1f}%  {k}")
    lines.append(f"#  total {tot / 1e6:.3f} ms")
    return lines

if __name__ == "__main__":
    out = []
    for rep in sys.argv[2:]:
        out += rep_summary(rep)
    if sys.argv[1] != "-":
        out += [""] + launch_summary(sys.argv[1])
    print("\n".join(out))
