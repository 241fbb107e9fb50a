"""Average DRAM traffic per k_far launch of one config-2 bench step, from the
ncu launch list (gpurun_out/launches.csv with dram__bytes_{read,write}.sum),
next to the algorithmic bytes of the same launches (the Z2 tile read + write,
32 m bytes per far row per shift per pass, plus the W rows a pass reads).
Writes profiles/r1_far_traffic.json, which bench.py reports as roofline.traffic.
(Experiment tooling, not part of the product.)"""
import csv, json, sys
from collections import defaultdict

def far_launches(n=4000, m=10, p=10, s=1000, nb=128, pw=128):
    """(rows, ncols_of_pass, w22) per far-kernel launch, mirroring
    enqueue_part's paired two-level loop (mode 0: far rows start at 0;
    pw = pass width: 128 on k_far4 for m = 10, 64 on k_far)."""
    ptop, out = p, []
    def far(rlo, r0, ncols):
        for jb in range(0, ncols, pw):
            out.append((r0 - rlo, min(pw, ncols - jb), jb == 0))
    ko = n
    while ko >= m + 1:
        nba = min(nb, ko - m)
        r0a = ptop + ko - nba
        kb = ko - nba
        if kb - m >= nb:
            r0b = r0a - nb
            far(r0b, r0a, nba)
            far(0, r0b, nb + nba)
            ko = kb - nb
        else:
            far(0, r0a, nba)
            ko = kb
    return out

def main(path="gpurun_out/launches.csv", dst="profiles/r1_far_traffic.json"):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hdr_i]
    iid, ik, imn, iv = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    per = defaultdict(dict)
    names = {}
    for r in rows[hdr_i + 1:]:
        if len(r) <= iv or not r[iid].isdigit():
            continue
        per[int(r[iid])][r[imn]] = float(r[iv].replace(",", ""))
        names[int(r[iid])] = r[ik]
    far_ids = sorted(i for i in per if "k_far" in names[i])
    m, s = 10, 1000
    geo = far_launches()
    if len(geo) != len(far_ids):
        print(f"warning: {len(far_ids)} k_far launches in the list, {len(geo)} expected", file=sys.stderr)
    k = min(len(geo), len(far_ids))
    dram = [per[i].get("dram__bytes_read.sum", 0) + per[i].get("dram__bytes_write.sum", 0) for i in far_ids[:k]]
    dur = [per[i].get("gpu__time_duration.sum", 0) for i in far_ids[:k]]
    alg = [rows_ * s * (32 * m) + s * (nc + (m if w22 else 0)) * m * 16 for rows_, nc, w22 in geo[:k]]
    out = {
        "what": "every k_far launch of one config-2 bench step (ncu launch list, "
                "--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum, "
                "--clock-control none; cold-cache, serialised)",
        "command": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                   "--clock-control none -k regex:k_ --csv python bench.py --profile --steps 1 --warmup 1",
        "launches": k,
        "dram_bytes_per_launch": sum(dram) / k,
        "algorithmic_bytes_per_launch": sum(alg) / k,
        "mean_duration_us": sum(dur) / k / 1e3,
        "note": "DRAM traffic vs the algorithmic Z2 stream (read + write of 32 m bytes per far "
                "row per shift per pass) + the W rows: no wasted re-reads; the kernel is "
                "FP64-bound (AI ~ 8 flop/B per pass)",
    }
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out, indent=1))

if __name__ == "__main__":
    main(*sys.argv[1:])
