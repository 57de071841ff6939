"""Render BASELINE.md §5 "Measured results" from bench.py JSON lines.

    python tools/render_baseline.py profiles/r02a/bench.json [more bench lines ...] [--write BASELINE.md]

Each argument is a file holding bench.py output (the last JSON line is used).  The headline line
gives the C2 table (per job, with the per-job ncu columns when present) and its c3 / c4 / c5
sub-records; a `--workload c1` line adds the C1 row; lines with n_gpus > 1 add scaling rows.
Without --write the section is printed.
"""
import argparse
import json
import os
import re

BEGIN = "<!-- measured:begin (tools/render_baseline.py) -->"
END = "<!-- measured:end -->"


def last_line(path):
    for ln in reversed(open(path).read().strip().splitlines()):
        if ln.startswith("{"):
            return json.loads(ln)
    raise SystemExit("no JSON line in " + path)


ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PEAK, NOMINAL = 6556.8, 8000.0


def ncu_fill(rows, workload, peak=None):
    """Set the committed per-job ncu numbers (profiles/ncu_jobs_<w>.json, the latest per-job launch
    lists) on every row, as a percentage of the line's own measured peak (PEAK if not given)."""
    peak = peak or PEAK
    p = os.path.join(ROOT, "profiles", "ncu_jobs_%s.json" % workload)
    if not os.path.exists(p):
        return
    m = {(j["N"], j["sign"]): j for j in json.load(open(p))["jobs"]}
    for r in rows:
        j = m.get((r["N"], r["sign"]))
        if j:
            r.update({"ncu_us": j["us"], "ncu_dram_GBs": j["dram_GBs"], "ncu_dram_bytes_per_elt": j["dram_bytes_per_elt"],
                      "pct_peak_measured": round(100 * j["dram_GBs"] / peak, 1),
                      "pct_peak_nominal": round(100 * j["dram_GBs"] / NOMINAL, 1)})


def fmt(v, nd=1):
    return "—" if v is None else ("%.*f" % (nd, v))


def render(lines, sources):
    out = [BEGIN, ""]
    head = [d for d in lines if d.get("n_gpus", 1) == 1 and "C2" in d["config"]["workload"]]
    for d, src in zip(lines, sources):
        if d is not (head[0] if head else None):
            continue
        c = d["clocks"]
        rl = d["roofline"]
        out += ["**Headline (C2, one B200)** — `%s`: **%.0f GFLOP/s** (std %.0f over %d rounds), %.3f ms per step; "
                "dominant kernel %s at %.0f GB/s = **%.3f** of the measured %.0f GB/s copy peak; SM clock %s MHz "
                "(max %s), throttle reasons %s." % (src, d["value"], d.get("value_std", 0), d.get("rounds", d["steps"]),
                                                     d["ms_per_step"], rl["kernel"].split(" ")[0], rl["achieved"],
                                                     rl["frac"], rl["peak"], c.get("sm_mhz"), c.get("sm_max_mhz"),
                                                     c.get("reasons") or "none"),
                ""]
        e = d.get("e2e") or {}
        cb = d.get("cpu_baseline") or {}
        out += ["End to end through `fftc_execute_host` (pinned host buffers, PCIe): %s GFLOP/s. Oracle (fp64 O2, "
                "%s cores, %s): %s GFLOP/s on a bounded sample (reported baseline only)." %
                (fmt(e.get("value")), cb.get("cores"), cb.get("cpu_model"), fmt(cb.get("value"), 2)), ""]
        ncu_fill(d["per_job"], "c2", rl["peak"])
        out += ["| N | sign | batch | µs (mean / median / p90) | GFLOP/s | eff. GB/s | ncu µs | ncu DRAM GB/s | %% of %.0f | "
                "%% of 8000 | plan |" % rl["peak"], "|---|---|---|---|---|---|---|---|---|---|---|"]
        for j in d["per_job"]:
            kern = re.search(r"kernel=(\S+)", j["plan"])
            out.append("| %d | %+d | %d | %.1f / %.1f / %.1f | %.0f | %.0f | %s | %s | %s | %s | %s |" % (
                j["N"], j["sign"], j["batch"], j["us"], j["us_median"], j["us_p90"], j["gflops"], j["eff_GBs"],
                fmt(j.get("ncu_us")), fmt(j.get("ncu_dram_GBs"), 0), fmt(j.get("pct_peak_measured")),
                fmt(j.get("pct_peak_nominal")), "`%s`" % kern.group(1) if kern else ""))
        out.append("")
        for w, title, bpe in (("c3", "C3 mixed radix", 16), ("c4", "C4 large N (two-pass bound: 32 B/element)", 32)):
            r = d.get(w)
            if not r or "jobs" not in r:
                continue
            ncu_fill(r["jobs"], w, rl["peak"])
            out += ["**%s** — %.0f GFLOP/s; fraction of the §8(d) bound (%d B per element): min %.3f." %
                    (title, r["value"], bpe, r["frac_min"]), "",
                    "| N | sign | µs | GFLOP/s | HBM passes | frac (§8(d) bound) | ncu DRAM GB/s | ncu B/element |",
                    "|---|---|---|---|---|---|---|---|"]
            for j in r["jobs"]:
                out.append("| %d | %+d | %.1f | %.0f | %d | %.3f | %s | %s |" % (
                    j["N"], j["sign"], j["us"], j["gflops"], j["hbm_passes"], j["frac"], fmt(j.get("ncu_dram_GBs"), 0),
                    fmt(j.get("ncu_dram_bytes_per_elt"), 2)))
            out.append("")
    for d, src in zip(lines, sources):
        if "C1" in d["config"]["workload"]:
            g = d.get("graph") or {}
            out += ["**C1** (N = 64 × 4096, launch-bound) — `%s`: %.0f GFLOP/s eager (L2 flushed between steps), "
                    "%s GFLOP/s as a CUDA graph." % (src, d["value"], fmt(g.get("value"), 0)), ""]
    multi = [(d, s) for d, s in zip(lines, sources) if d.get("n_gpus", 1) > 1]
    if multi:
        out += ["| GPUs | value GFLOP/s | ms per step | scaling | gpus active | c5 six-step (ms, variants) | source |",
                "|---|---|---|---|---|---|---|"]
        for d, s in multi:
            c5 = d.get("c5") or {}
            v = ", ".join("%s %.2f" % (x["exchange"], x["ms"]) for x in c5.get("variants", [])) or c5.get("error", "—")
            out.append("| %d | %.0f | %.3f | %s | %s | %s | `%s` |" % (d["n_gpus"], d["value"], d["ms_per_step"],
                                                                      d["scaling"],
                                                                      (d.get("multi_gpu") or {}).get("gpus_active"),
                                                                      v, s))
        out.append("")
    out.append(END)
    return "\n".join(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("files", nargs="+")
    ap.add_argument("--write")
    a = ap.parse_args()
    lines = [last_line(f) for f in a.files]
    txt = render(lines, a.files)
    if not a.write:
        print(txt)
        return
    doc = open(a.write).read()
    if BEGIN in doc:
        doc = doc[:doc.index(BEGIN)] + txt + doc[doc.index(END) + len(END):]
    else:
        i = doc.index("## 5. Measured results")
        j = doc.find("\n## ", i + 5)
        body = "## 5. Measured results\n\nRendered by `tools/render_baseline.py` from the committed bench lines.\n\n" + txt + "\n"
        doc = doc[:i] + body + (doc[j:] if j > 0 else "")
    open(a.write, "w").write(doc)


if __name__ == "__main__":
    main()
