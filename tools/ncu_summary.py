"""Summarise an ncu launch list (CSV from `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv --log-file ...`) into per-kernel rows and the bench traffic file.

    python tools/ncu_summary.py launches.csv [--traffic profiles/traffic_c2.json] [--md out.md]
"""
import argparse
import csv
import json
import statistics
from collections import OrderedDict, defaultdict


def parse(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hdr]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    launches = OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        d = launches.setdefault(int(r[ii]), {"kernel": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", ""))
    return list(launches.values())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--traffic")
    ap.add_argument("--md")
    ap.add_argument("--kernel", default="k_fused_batch")
    a = ap.parse_args()
    L = parse(a.csv)
    by = defaultdict(list)
    for d in L:
        by[d["kernel"]].append(d)
    tot = sum(d.get("gpu__time_duration.sum", 0) for d in L)
    lines = ["| kernel | launches | mean us | share of time | mean DRAM bytes | DRAM GB/s |", "|---|---|---|---|---|---|"]
    for k, ds in sorted(by.items(), key=lambda kv: -sum(x.get("gpu__time_duration.sum", 0) for x in kv[1])):
        t = [x.get("gpu__time_duration.sum", 0) for x in ds]
        b = [x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in ds]
        mt, mb = statistics.mean(t), statistics.mean(b)
        lines.append("| `%s` | %d | %.1f | %.1f%% | %.3e | %.0f |" % (k[:90], len(ds), mt / 1e3, 100 * sum(t) / tot,
                                                                    mb, mb / mt if mt else 0))
    md = "\n".join(lines)
    print(md)
    if a.md:
        open(a.md, "w").write(md + "\n")
    if a.traffic:
        sel = [d for d in L if a.kernel in d["kernel"]]
        b = statistics.mean(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in sel)
        t = statistics.mean(d["gpu__time_duration.sum"] for d in sel)
        json.dump({"source": a.csv, "kernel": a.kernel, "launches": len(sel), "dram_bytes_per_launch": b,
                   "ncu_mean_duration_ns": t, "share_of_step_time": sum(d["gpu__time_duration.sum"] for d in sel) / tot},
                  open(a.traffic, "w"), indent=1)


if __name__ == "__main__":
    main()
