"""Print the key numbers of one or more bench.py JSON lines (log files)."""
import json
import sys

for path in sys.argv[1:]:
    lines = [l for l in open(path).read().strip().splitlines() if l.startswith("{")]
    if not lines:
        print(path, "no JSON line")
        continue
    d = json.loads(lines[-1])
    print(path)
    print("  value", round(d["value"], 1), "ms/step", round(d["ms_per_step"], 1),
          "peak_gb", round(d["peak_gb_per_gpu"], 2), "frac", round(d["roofline"]["frac"] or 0, 3),
          "e2e", d["e2e"] and round(d["e2e"]["value"], 1), "clk", d["clocks"].get("sm_mhz"))
    for k, v in d["kernels"].items():
        print(f"    {k:10s} {v['ms_per_step']:8.1f} ms  {v['launches_per_step']}")
