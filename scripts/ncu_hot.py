"""Top warp-stall SASS lines of one kernel from `ncu --page source --csv --print-source sass`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = None; data = []
for r in rows:
    if "Address" in r and "Source" in r:
        hdr = r; continue
    if hdr and len(r) == len(hdr) and r[0].startswith("0x"):
        data.append(r)
ia, isrc = hdr.index("Address"), hdr.index("Source")
iss = hdr.index("Warp Stall Sampling (All Samples)")
ins = hdr.index("Warp Stall Sampling (Not-issued Samples)")
v = lambda r, i: int(r[i] or 0)
tot = sum(v(r, iss) for r in data)
print("total samples", tot)
for r in sorted(data, key=lambda r: -v(r, iss))[:n]:
    print(f"{v(r,iss):6d} {v(r,ins):6d} {100*v(r,iss)/max(tot,1):5.1f}% {r[ia][-5:]} {r[isrc].strip()[:90]}")
