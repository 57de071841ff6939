"""Per-job ncu numbers for a bench workload (HBM GB/s from ncu per config).

    # on the GPU box, under ncu (each job runs exactly once, in bench.py's job order):
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file gpurun_out/X/jobs_c2.csv \
        python tools/ncu_jobs.py run --workload c2 --map gpurun_out/X/jobs_c2_map.json
    # here: launch list + job map -> profiles/ncu_jobs_c2.json (read by bench.py per_job)
    python tools/ncu_jobs.py parse gpurun_out/X/jobs_c2.csv gpurun_out/X/jobs_c2_map.json \
        --out profiles/ncu_jobs_c2.json --source profiles/r02/jobs_c2.csv

`dram_GBs` = (dram__bytes_read.sum + dram__bytes_write.sum) / gpu__time_duration.sum summed
over the job's launches (ncu replays each kernel with caches flushed: cold-cache, serialised).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def run(a):
    import torch
    import bench
    desc, jobs = bench.workloads(a.workload)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    js = bench.JobSet(jobs, dev, 0, 1)
    stream = torch.cuda.current_stream(dev)
    js.run(stream)
    torch.cuda.synchronize(dev)
    m = [{"N": N, "batch": b1 - b0, "sign": s, "launches": js.plans[i].launches(), "plan": js.plans[i].describe()}
         for i, (N, B, s, d, b0, b1) in enumerate(js.jobs)]
    json.dump({"workload": a.workload, "desc": desc, "jobs": m}, open(a.map, "w"), indent=1)
    js.close()


def parse(a):
    from ncu_summary import parse as parse_csv
    L = parse_csv(a.csv)
    m = json.load(open(a.map))
    need = sum(j["launches"] for j in m["jobs"])
    if len(L) < need:
        raise SystemExit("launch list has %d launches, the job map needs %d" % (len(L), need))
    out, i = [], 0
    for j in m["jobs"]:
        ls = L[i:i + j["launches"]]
        i += j["launches"]
        t = sum(x["gpu__time_duration.sum"] for x in ls)  # ns
        b = sum(x["dram__bytes_read.sum"] + x["dram__bytes_write.sum"] for x in ls)
        e = j["N"] * j["batch"]
        out.append({"N": j["N"], "sign": j["sign"], "batch": j["batch"], "launches": j["launches"],
                    "kernels": sorted({x["kernel"].split("(")[0][:60] for x in ls}),
                    "us": round(t / 1e3, 2), "dram_bytes": b, "dram_GBs": round(b / t, 1),
                    "dram_bytes_per_elt": round(b / e, 3)})
    json.dump({"workload": m["workload"], "source": a.source or a.csv,
               "how": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                      "--clock-control none; one execute per job (tools/ncu_jobs.py)",
               "jobs": out}, open(a.out, "w"), indent=1)
    for r in out:
        print("N=%-8d sign=%+d  %8.1f us  %7.1f GB/s  %.2f B/elt" % (r["N"], r["sign"], r["us"], r["dram_GBs"],
                                                                  r["dram_bytes_per_elt"]))


def main():
    ap = argparse.ArgumentParser()
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run")
    r.add_argument("--workload", default="c2")
    r.add_argument("--map", required=True)
    p = sub.add_parser("parse")
    p.add_argument("csv")
    p.add_argument("map")
    p.add_argument("--out", required=True)
    p.add_argument("--source")
    a = ap.parse_args()
    run(a) if a.cmd == "run" else parse(a)


if __name__ == "__main__":
    main()
