"""Per-kernel summary of an `ncu --set full` report (CSV raw page on stdin or
file): duration, tensor-pipe activity, issue activity, DRAM bytes and
throughput, pipe utilisation, top stall reasons. Used to write profiles/."""
import csv, re, sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[0], rows[2:]
units = rows[1]
col = {h: i for i, h in enumerate(hdr)}

def val(d, k):
    try:
        return float(d[col[k]])
    except (KeyError, ValueError):
        return None

def name(d):
    n = d[col["Kernel Name"]]
    m = re.search(r"Epi\w+", n)
    base = re.sub(r"\(.*", "", n).split("::")[-1]
    cg = re.search(r"\(int\)(\d)>\(CUtensorMap", n)
    return (f"gemm_kernel<{m.group(0)}>" + (" 2-SM" if cg and cg.group(1) == "2" else "")) if m else base

stall = [h for h in hdr if re.match(r"smsp__average_warps_issue_stalled_.*_per_issue_active.ratio", h)]
pipes = [h for h in hdr if re.match(r"sm__inst_executed_pipe_(xu|alu|fma|lsu|fp64).avg.pct_of_peak_sustained_active", h)]
print(f"{'kernel':34s} {'dur':>9s} {'tensor%':>8s} {'issue%':>7s} {'DRAM GB':>8s} {'DRAM%':>6s} {'SMclk':>6s}  pipes / top stalls")
for d in data:
    dur = val(d, "gpu__time_duration.sum")
    du = units[col["gpu__time_duration.sum"]]
    rd = (val(d, "dram__bytes_read.sum") or 0) + (val(d, "dram__bytes_write.sum") or 0)
    bu = units[col["dram__bytes_read.sum"]]
    scale = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}.get(bu, 1.0)
    tp = val(d, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active") or 0
    st = sorted(((val(d, h) or 0, h.split("stalled_")[1].split("_per")[0]) for h in stall), reverse=True)[:3]
    pp = " ".join(f"{h.split('pipe_')[1][:4]}{(val(d, h) or 0):.0f}" for h in pipes)
    print(f"{name(d):34s} {dur:8.1f}{du[:2]:>2s} {tp:8.1f} {val(d, 'sm__issue_active.avg.pct_of_peak_sustained_elapsed') or 0:7.1f} "
          f"{rd * scale:8.3f} {val(d, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed') or 0:6.1f} "
          f"{(val(d, 'sm__cycles_elapsed.avg.per_second') or 0):6.2f}  {pp} | " + ", ".join(f"{n}={v:.2f}" for v, n in st))
