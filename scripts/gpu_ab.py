"""Same-box A/B: run bench.py (c4, device path) under several env configs,
interleaved over repetitions, and print one summary line per run plus the
per-config median ms/step."""
import json, os, statistics, subprocess, sys

cfgs = [c for c in os.environ.get("AB_CFGS", "SWTB_PARTS=2").split(";") if c.strip()]
reps = int(os.environ.get("AB_REPS", "2"))
res = {c: [] for c in cfgs}
os.makedirs("gpurun_out", exist_ok=True)
for r in range(reps):
    for c in cfgs:
        env = dict(os.environ)
        for kv in c.split():
            k, v = kv.split("=", 1)
            env[k] = v
        out = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3",
                              "--no-cpu-baseline", "--no-e2e"] + sys.argv[1:],
                             env=env, capture_output=True, text=True, timeout=900)
        line = [l for l in out.stdout.splitlines() if l.startswith("{")]
        if not line:
            print("FAILED", c, out.stderr[-2000:]); continue
        d = json.loads(line[-1])
        res[c].append(d["ms_per_step"])
        k = d["kernels"]
        print(f"[{r}] {c:40s} {d['ms_per_step']:7.1f} ms  clk {d['clocks'].get('sm_mhz')}  " +
              " ".join(f"{n}={v['ms_per_step']:.0f}" for n, v in k.items() if v['ms_per_step'] > 0), flush=True)
for c in cfgs:
    if res[c]:
        print(f"MEDIAN {c:40s} {statistics.median(res[c]):7.1f} ms/step over {len(res[c])}")
