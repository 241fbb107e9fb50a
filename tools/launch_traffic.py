"""Per-launch DRAM traffic of one kernel family from an ncu launch list
(--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,
--csv), merged into profiles/r2_far_traffic.json under key cfg<N>; bench.py
reports it as roofline.traffic.  (Experiment tooling, not part of the product.)

    python tools/launch_traffic.py gpurun_out/launches.csv k_fark 4 [dst.json]
"""
import csv
import json
import os
import re
import sys
from collections import defaultdict


def per_launch(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hdr_i]
    iid, ik, imn, iv = (h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"),
                        h.index("Metric Value"))
    per, names = defaultdict(dict), {}
    for r in rows[hdr_i + 1:]:
        if len(r) <= iv or not r[iid].isdigit():
            continue
        per[int(r[iid])][r[imn]] = float(r[iv].replace(",", ""))
        names[int(r[iid])] = r[ik]
    return per, names


def main(path, kernel, cfg, dst="profiles/r2_far_traffic.json"):
    per, names = per_launch(path)
    ids = sorted(i for i in per if re.search(kernel, names[i]))
    if not ids:
        sys.exit(f"no launch of {kernel!r} in {path}")
    dram = [per[i].get("dram__bytes_read.sum", 0) + per[i].get("dram__bytes_write.sum", 0)
            for i in ids]
    dur = [per[i].get("gpu__time_duration.sum", 0) for i in ids]
    tot = sum(v.get("gpu__time_duration.sum", 0) for v in per.values())
    rec = {
        "what": f"every {kernel} launch of one config-{cfg} bench step (ncu launch list, "
                "--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                "--clock-control none; cold-cache, serialised)",
        "launches": len(ids),
        "dram_bytes_per_launch": sum(dram) / len(ids),
        "mean_duration_us": sum(dur) / len(ids) / 1e3,
        "share_of_listed_time": sum(dur) / tot if tot else None,
        "kernel_names": sorted({names[i][:90] for i in ids}),
    }
    out = json.load(open(dst)) if os.path.exists(dst) else {}
    out[f"cfg{cfg}"] = rec
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(rec, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]), *sys.argv[4:])
