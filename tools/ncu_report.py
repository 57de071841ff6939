"""Key metrics per kernel launch from an ncu --set full report (reads `ncu -i --page raw --csv`).
    python tools/ncu_report.py gpurun_out/prof_a.ncu-rep [--every 2]"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "us", 1e-3),
    ("dram__bytes_read.sum", "rdMB", 1e-6),
    ("dram__bytes_write.sum", "wrMB", 1e-6),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%", 1),
    ("launch__registers_per_thread", "regs", 1),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%", 1),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1%", 1),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "bankc", 1e-6),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shwf", 1e-6),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "l2rdsec", 1e-6),
]
STALLS = ["long_scoreboard", "barrier", "mio_throttle", "short_scoreboard", "lg_throttle", "not_selected",
          "selected", "wait", "math_pipe_throttle", "drain", "no_instruction", "branch_resolving", "membar"]


def main():
    rep = sys.argv[1]
    every = int(sys.argv[sys.argv.index("--every") + 1]) if "--every" in sys.argv else 1
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    idx = {n: i for i, n in enumerate(h)}
    ki = idx["Kernel Name"]
    for n, r in enumerate(rows[2:]):
        if n % every != every - 1:
            continue
        name = r[ki]
        name = name[name.find("Sched<") + 6:name.find(">")] if "Sched<" in name else name[:40]
        vals = []
        for k, lab, sc in KEYS:
            v = r[idx[k]].replace(",", "") if k in idx else ""
            try:
                vals.append("%s=%.1f" % (lab, float(v) * sc))
            except ValueError:
                vals.append("%s=?" % lab)
        st = []
        for s in STALLS:
            k = "smsp__pcsamp_warps_issue_stalled_" + s
            if k in idx:
                try:
                    st.append((float(r[idx[k]].replace(",", "")), s))
                except ValueError:
                    pass
        tot = sum(v for v, _ in st) or 1
        st.sort(reverse=True)
        print("%-28s %s" % (name[:28], " ".join(vals)))
        print("%28s stalls: %s" % ("", " ".join("%s=%.0f%%" % (s, 100 * v / tot) for v, s in st[:6])))


if __name__ == "__main__":
    main()
