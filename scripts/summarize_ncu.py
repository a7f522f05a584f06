"""Summarise ncu outputs (gpurun_out/) into profiles/: the per-kernel share of
the launch list (gpu__time_duration.sum, cold-cache and serialised) and the key
counters of a --set full capture, plus profiles/ncu_traffic.json that bench.py
reads for roofline.traffic (dram read+write bytes per launch)."""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launch_shares(path):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    agg = defaultdict(lambda: [0, 0.0])
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "").strip()
        agg[name][0] += 1
        agg[name][1] += float(r["Metric Value"].replace(",", "")) * scale[r["Metric Unit"]]
    tot = sum(a[1] for a in agg.values())
    return [(k, c, us, 100 * us / tot) for k, (c, us) in sorted(agg.items(), key=lambda x: -x[1][1])], tot


def full_counters(rep):
    # a .ncu-rep (read with ncu -i) or its "--page raw --csv" export
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
            "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "lts__t_bytes.sum", "l1tex__t_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "l1tex__throughput.avg.pct_of_peak_sustained_active",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
    res = []
    for v in rows[2:]:
        res.append({x: (v[i], u[i]) for i, x in enumerate(h) if x in want})
    return res


def to_bytes(val, unit):
    f = float(val.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def main():
    tag, cfg, launches, rep, key = sys.argv[1:6]  # e.g. r01 C4 gpurun_out/launches_C4.csv gpurun_out/prof.ncu-rep restrict
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    shares, tot = launch_shares(launches)
    lines = [f"# ncu launch list ({cfg}, {tag}): gpu__time_duration.sum, --clock-control none",
             "# cold-cache serialised launches: compare SHARES, not absolute times", "",
             f"{'kernel':32s} {'launches':>8s} {'total_us':>12s} {'share':>7s}"]
    lines += [f"{k:32s} {c:8d} {us:12.1f} {pct:6.1f}%" for k, c, us, pct in shares]
    lines.append(f"{'TOTAL':32s} {'':8s} {tot:12.1f}")
    open(os.path.join(prof, f"{tag}_{cfg}_launches.txt"), "w").write("\n".join(lines) + "\n")
    counters = full_counters(rep)
    open(os.path.join(prof, f"{tag}_{cfg}_{key}_ncu_full.json"), "w").write(json.dumps(counters, indent=1))
    c = counters[0]
    traffic = to_bytes(*c["dram__bytes_read.sum"]) + to_bytes(*c["dram__bytes_write.sum"])
    tpath = os.path.join(prof, "ncu_traffic.json")
    t = json.load(open(tpath)) if os.path.exists(tpath) else {}
    t.setdefault(cfg, {})[key] = traffic
    json.dump(t, open(tpath, "w"), indent=1, sort_keys=True)
    print("\n".join(lines))
    print(json.dumps(c, indent=1))
    print("traffic bytes/launch", traffic)


if __name__ == "__main__":
    main()
