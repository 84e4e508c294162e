"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel-family total time, share of the step and launch count."""
import csv, re, sys, collections

def family(name):
    m = re.search(r"(Epi\w+?)<", name) or re.search(r"(Epi\w+)", name)
    base = re.sub(r"\(.*", "", name).split("::")[-1]
    base = re.sub(r"<.*", "", base)
    if "gemm_kernel" in name and m:
        split = re.search(r",\s*(\d)>\(", name)
        return f"gemm_kernel<{m.group(1)}>" + (f" split{split.group(1)}" if split else "")
    return base

lines = [l for l in open(sys.argv[1]) if l.startswith("\"")]
rows = list(csv.DictReader(lines))
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in rows:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    f = family(r["Kernel Name"])
    tot[f] += float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else 1e3 if r["Metric Unit"] == "ms" else 1)
    cnt[f] += 1
all_us = sum(tot.values())
print(f"{'kernel':48s} {'launches':>8s} {'total ms':>10s} {'share':>7s} {'us/launch':>10s}")
for f, t in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{f:48s} {cnt[f]:8d} {t/1e3:10.2f} {100*t/all_us:6.1f}% {t/cnt[f]:10.1f}")
print(f"{'TOTAL':48s} {sum(cnt.values()):8d} {all_us/1e3:10.2f}")
