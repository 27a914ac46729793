"""One line per bench.py JSON output file: config, ms/step, roofline frac, clocks, e2e, value.
    python tools/bench_summary.py gpurun_out/b_*.json"""
import json
import sys

for path in sys.argv[1:]:
    try:
        d = json.loads(open(path).read().strip().splitlines()[-1])
    except Exception as e:   # noqa: BLE001
        print(path, "unreadable:", e)
        continue
    if d.get("impl") == "reference":
        print(path, "reference", d["config"]["workload"], "value %.2f" % d["value"], d["cpu_baseline"]["kind"],
              "cores", d["cpu_baseline"]["cores"], "port", d.get("port", {}).get("value"))
        continue
    print(path, d["config"]["workload"], "ms %.4f" % d["ms_per_step"], "frac %.4f" % d["roofline"]["frac"],
          "value %.1f" % d["value"], "e2e %.1f" % d["e2e"]["value"], "clk", d["clocks"].get("sm_mhz"),
          d["clocks"].get("reasons"), "samples", d["clocks"].get("samples"),
          "verified", d.get("verified_images_vs_oracle"))
