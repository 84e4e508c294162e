"""DRAM traffic per output-layer GEMM kind from an `ncu --set full` raw CSV
export (argv[1]) -> profiles/r01_ncu_traffic.json format (argv[2]); bench.py
multiplies each kind's achieved DRAM rate by its live duration."""
import csv, json, re, sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
tscale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}
out = {}
for d in data:
    m = re.search(r"(EpiFwdLse|EpiBwdDh|EpiDzGate|EpiAtomic)", d[col["Kernel Name"]])
    if not m:
        continue
    k = m.group(1)
    b = sum(float(d[col[n]]) * scale.get(units[col[n]], 1.0)
            for n in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    t = float(d[col["gpu__time_duration.sum"]]) * tscale.get(units[col["gpu__time_duration.sum"]], 1e-6)
    e = out.setdefault(k, {"launches": 0, "dram_bytes": 0.0, "seconds": 0.0})
    e["launches"] += 1
    e["dram_bytes"] += b
    e["seconds"] += t
for e in out.values():
    e["dram_bytes_per_launch"] = e["dram_bytes"] / e["launches"]
    e["achieved_dram_GBps"] = e["dram_bytes"] / e["seconds"] / 1e9
json.dump({"source": "ncu --set full --clock-control none of the timed bench.py c4 step "
                     "(NVTX range 'timed'; the ncu_full_c4_summary.txt of the same round); EpiAtomic = "
                     "the dW_O+db_O GEMM (EpiAtomicDb)", "kernels": out},
          open(sys.argv[2], "w"), indent=1)
print(json.dumps(out, indent=1))
