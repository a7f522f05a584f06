"""Summarise ncu --set full captures of the setup contractions (raw csv pages of
gpurun_out/prof_setup_{dmma,ffma}): duration, DRAM bytes, FP64 tensor (DMMA)
and FP64 FMA pipe utilisation per launch.
usage: python scripts/summarize_setup_ncu.py gpurun_out/prof_setup_dmma.raw.csv ... > profiles/..."""
import csv
import json
import sys

KEYS = {
    "time": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "dmma_pipe_pct_active": "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct_active": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_clock": "sm__cycles_elapsed.avg.per_second",
}
out = []
for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        e = {"capture": path.split("/")[-1], "kernel": d["Kernel Name"]}
        for k, m in KEYS.items():
            v = d.get(m)
            if v in (None, ""):
                continue
            v = float(v.replace(",", ""))
            unit = u.get(m, "")
            e[k] = round(v, 3)
            if unit and not k.endswith("pct_active") and k != "dram_pct":
                e[k + "_unit"] = unit
        out.append(e)
print(json.dumps(out, indent=1))
