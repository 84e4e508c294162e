"""Top warp-stall-sampled SASS instructions of the first kernel in an
`ncu --page source --csv --print-source sass` export (argv[1])."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_n = hdr.index("Warp Stall Sampling (Not-issued Samples)")
i_src = hdr.index("Source")
data = []
for r in rows[2:]:
    if len(r) < len(hdr):
        break  # next kernel
    data.append((int(r[i_s] or 0), int(r[i_n] or 0), r[i_src].strip()))
tot = sum(d[0] for d in data)
print("samples", tot, "instructions", len(data))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
top = sorted(range(len(data)), key=lambda k: -data[k][0])[:n]
for k in sorted(top):
    print(f"{k:5d} {data[k][0]:6d} {100.0 * data[k][0] / tot:5.1f}%  {data[k][2][:100]}")
