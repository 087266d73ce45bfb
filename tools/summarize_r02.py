"""Reduce the round-2 ncu CSVs in gpurun_out/ to profiles/streaming_r02.json
(per kernel: launches, mean duration, DRAM bytes per launch, ncu DRAM
throughput %, achieved DRAM GB/s and its fraction of the measured peak) and
profiles/launch_shares_r02.json (per-kernel totals of the bench launch list)."""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
O = os.path.join(ROOT, "gpurun_out")
PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6546.9


def metrics(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, collections.OrderedDict()
    for r in rows:
        if len(r) > 5 and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            out.setdefault(int(d["ID"]), {"kernel": d["Kernel Name"].split("(")[0]})[d["Metric Name"]] = float(
                d["Metric Value"].replace(",", ""))
    return list(out.values())


def summarize(path, label):
    per = collections.OrderedDict()
    for m in metrics(path):
        per.setdefault(m["kernel"], []).append(m)
    res = {}
    for k, ms in per.items():
        dur = sum(x["gpu__time_duration.sum"] for x in ms) / len(ms)  # ns
        rd = sum(x.get("dram__bytes_read.sum", 0) for x in ms) / len(ms)
        wr = sum(x.get("dram__bytes_write.sum", 0) for x in ms) / len(ms)
        gbs = (rd + wr) / dur  # bytes per ns = GB/s
        res[k] = {"launches": len(ms), "mean_us": round(dur / 1e3, 2), "dram_read_bytes": int(rd),
                  "dram_write_bytes": int(wr),
                  "ncu_dram_throughput_pct": round(sum(x["dram__throughput.avg.pct_of_peak_sustained_elapsed"]
                                                       for x in ms) / len(ms), 2),
                  "dram_gbs": round(gbs, 1), "frac_of_measured_peak": round(gbs / PEAK, 3)}
    return {label: res}


out = {"peak_gbs": PEAK, "source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
       "dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none "
       "(cold, serialised launches; tools/capture_profiles_r02.sh)"}
for f, label in (("build_kernels_r02_2m.csv", "build, 2M rows (device-resident)"),
                 ("build_kernels_r02_25m.csv", "build, 25M rows (device-resident)"),
                 ("fullscan_smallq_r02_2m.csv", "single-query full scan, N=2M"),
                 ("fullscan_smallq_r02_200m.csv", "single-query full scan, N=200M")):
    p = os.path.join(O, f)
    if os.path.exists(p):
        out.update(summarize(p, label))
json.dump(out, open(os.path.join(ROOT, "profiles", "streaming_r02.json"), "w"), indent=1)

p = os.path.join(O, "launches_r02_bench.csv")
if os.path.exists(p):
    tot = collections.defaultdict(lambda: [0, 0.0])
    for m in metrics(p):
        tot[m["kernel"]][0] += 1
        tot[m["kernel"]][1] += m["gpu__time_duration.sum"] / 1e3
    all_us = sum(t for _, t in tot.values())
    shares = {k: {"launches": c, "total_us": round(t, 1), "mean_us": round(t / c, 3),
                  "share": round(t / all_us, 4)} for k, (c, t) in sorted(tot.items(), key=lambda x: -x[1][1])}
    json.dump({"command": "python bench.py --steps 64 --warmup 64 --no-extras --cpu-budget-s 1 (under ncu, "
                          "-c 3000; includes 8 replica builds and the e2e leg)", "kernels": shares},
              open(os.path.join(ROOT, "profiles", "launch_shares_r02.json"), "w"), indent=1)
print(json.dumps(out, indent=1)[:3000])
