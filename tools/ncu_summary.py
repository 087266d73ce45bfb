"""Distil ncu reports into profiles/ (run here, after gpurun brought them back).

    python tools/ncu_summary.py gpurun_out/prof_query_r01.ncu-rep:k_query_w1 \
        gpurun_out/ncu_raw_fullscan_r01.csv:k_fullscan_w1 ... --launches gpurun_out/launches.csv

(each spec is an .ncu-rep or its exported `--page raw --csv` page; --update
replaces only the named kernels' entries of the existing summary)

Writes profiles/ncu_summary.json (per-kernel duration, DRAM bytes, issue and
occupancy figures; bench.py reads dram_bytes_per_launch as roofline.traffic)
and profiles/launch_shares.json (per-kernel share of the bench launch list).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "smsp__inst_executed.sum": "warp_instructions",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3,
         "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}


def raw(rep: str) -> dict:
    if rep.endswith(".csv"):  # an exported `--page raw --csv` page
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, u, v = r[0], r[1], r[2]
    return {k: (val, unit) for k, unit, val in zip(h, u, v)}


def main() -> None:
    args = sys.argv[1:]
    launches = None
    update = "--update" in args  # keep the other kernels' entries of the existing summary
    args = [a for a in args if a != "--update"]
    if "--launches" in args:
        i = args.index("--launches")
        launches = args[i + 1]
        args = args[:i] + args[i + 2:]
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summary = json.load(open(path)) if update and os.path.exists(path) else {}
    for spec in args:
        rep, name = spec.split(":")
        d = raw(rep)
        e = {"report": os.path.basename(rep), "kernel": d.get("Kernel Name", ("", ""))[0]}
        for k, short in KEYS.items():
            if k not in d:
                continue
            val, unit = d[k]
            try:
                x = float(val.replace(",", ""))
            except ValueError:
                continue
            if short == "duration":
                e["duration_us"] = x * SCALE.get(unit, 1)
            elif short.startswith("dram_r") or short.startswith("dram_w"):
                e[short + "_bytes"] = x * SCALE.get(unit, 1)
            else:
                e[short] = x
        e["dram_bytes_per_launch"] = e.get("dram_read_bytes", 0) + e.get("dram_write_bytes", 0)
        summary[name] = e
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(path, "w") as f:
        json.dump(summary, f, indent=1)
    if launches:
        rows = list(csv.reader(open(launches)))
        hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
        h = rows[hi]
        agg = {}
        for r in rows[hi + 1:]:
            d = dict(zip(h, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            nm = d["Kernel Name"].split("(")[0]
            us = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1)
            a = agg.setdefault(nm, [0, 0.0])
            a[0] += 1
            a[1] += us
        tot = sum(x[1] for x in agg.values())
        shares = {k: {"launches": c, "total_us": round(t, 2), "mean_us": round(t / c, 3),
                      "share": round(t / tot, 4)} for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])}
        with open(os.path.join(ROOT, "profiles", "launch_shares.json"), "w") as f:
            json.dump(shares, f, indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
