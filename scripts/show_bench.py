"""Summarise gpurun_out/bench_<cfg>.json lines (development helper)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.load(open(f"gpurun_out/bench_{f}.json"))
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable:", e)
        continue
    it = d["roofline"]["iteration"]
    print(f, d["value"], "iters", d["iterations_per_solve"], "ms/it", d["ms_per_iteration"], "iterfrac",
          it["frac"], it.get("cycle"), "e2e", d["e2e"]["value"], "clk", d["clocks"]["sm_mhz"])
    print("   ", {k: (v["avg_us"], round(v["gbs"])) for k, v in d["kernels"].items()})
