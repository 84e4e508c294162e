#!/usr/bin/env python
"""Benchmark: sample-wise transducer loss + all gradients on B200.

Workload (BASELINE.json metric, configs[3], the north star):
  B=1024 T=1000 U=200 V=1024 H=H_A=H_L=512, reference synth_inputs (seed 1,
  padding ramp), one step = loss + gradients for h^A, h^L, theta^J, theta^O
  over the whole batch. Under torchrun with N GPUs the fixed B=1024 batch is
  sharded by sample (b % N == rank) and theta-grads are summed with one NCCL
  all-reduce inside libswt_b200 (strong scaling).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c4|c3|c2|c1|c5] [--precision bf16|bf16x|tf32]

Prints ONE JSON line on rank 0. `value` = samples/s with inputs resident in
HBM (device pointers through the C ABI); `e2e` = the same call with pinned
HOST buffers, every step's h2d inputs and d2h gradients inside the timed
region. `roofline` is for the output-layer GEMM family (f^O forward,
recompute, dz, dW_O: >99% of algorithmic FLOPs), timed live with CUDA events
on the engine's stream; in the fp16 default the backward GEMMs walk only the
tiles whose fp16 dh is not exactly zero, so the family's
algorithmic work counts 2 H V flops per cell for the forward and 4 H V per
cell of the walked tiles, and `secondary.fp16_dense_backward` times the same
step with every tile. The reference arm times the unmodified reference CPU
engine (oracle/_ref, compiled from /root/reference) on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {  # name: (B, T, U, V, H)   (BASELINE.json "configs")
    "c1": (1, 50, 10, 32, 64),
    "c2": (32, 200, 50, 512, 256),
    "c3": (128, 500, 100, 1024, 512),
    "c4": (1024, 1000, 200, 1024, 512),
    "c5": (256, 750, 150, 4096, 640),
}
METRIC = "loss+grad samples/sec at B=1024,T=1000,U=200,V=1024; peak GB/GPU"
# per-GEMM-kind DRAM rates from the committed ncu --set full captures (the
# roofline's `traffic`): the stored-logits pipeline and the recompute one
TRAFFIC_STORED = None  # no capture of the opt-in stored-logits pipeline
TRAFFIC_RECOMPUTE = "r02_ncu_traffic.json"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["bf16_tflops"], p.get("bf16_tflops_sustained"), p["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


def algorithmic_flops(t_len, u_len, V, H, HA, HL, samples=None):
    idx = range(len(t_len)) if samples is None else samples
    out = joint = 0
    for b in idx:
        T, U1 = int(t_len[b]), int(u_len[b]) + 1
        out += 6 * T * U1 * H * V
        joint += 6 * H * (T * HA + U1 * HL)
    return out, joint


def memory_model(B, T, U, V, H, HA, HL, t_len, u_len):
    """The reference's analytic memory model (proj/core/src/engine.cpp:52-68,
    f32): the fully batched engine needs at least B x lattice_trio_bytes of
    the padded extents; the sample-wise (+PR) engine peaks at the inputs +
    outputs + the largest sample's working set. The batched comparator of
    SURVEY §8(f) row 1, reported analytically (it does not fit a B200)."""
    f32 = 4
    trio = lambda T_, U1_: T_ * U1_ * (H + 2 * V) * f32
    def working(T_, U1_):
        cells = T_ * U1_
        e = cells * (2 * H + 2 * V) + 3 * cells + (T_ + U1_) * H
        e += 2 * (T_ * HA + U1_ * HL) + H * (HA + HL + 1) + V * (H + 1)
        return e * f32
    io = (B * T * HA + B * (U + 1) * HL + H * (HA + HL + 1) + V * (H + 1)) * f32
    big = max(range(len(t_len)), key=lambda b: int(t_len[b]) * (int(u_len[b]) + 1))
    batched = B * trio(T, U + 1)
    return {"batched_engine_min_bytes": batched,
            "batched_fits_one_b200": batched < 180e9,
            "reference_sample_wise_pr_peak_bytes": 2 * io + working(int(t_len[big]), int(u_len[big]) + 1),
            "source": "reference engine.cpp:52-68 (lattice_trio_bytes, sample_working_bytes), f32"}


class Clocks:
    """nvidia-smi sampler running during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.rows = []
        if self.proc is None:
            return
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9:
                self.rows.append(f)

    def summary(self):
        rows = getattr(self, "rows", [])
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[1]) for r in rows if num(r[1])]
        pw = [num(r[3]) for r in rows if num(r[3])]
        pmax = max(pw) if pw else 0.0
        load = [s for s, p in zip(sm, pw) if p >= 0.5 * pmax] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9])
                          if v.lower() == "active"})
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": num(rows[0][2]), "reasons": reasons,
                "samples": len(rows), "power_w_max": max(pw) if pw else None}


# ---------------------------------------------------------------------------
# reference arm: the unmodified reference CPU engine on a bounded sample

def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# The reference arm's bounded sample (fixed, independent of --steps/--warmup):
# every sample at the config's full label extent U, vocabulary V and width H,
# with REF_T_SAMPLE frames (c4: 48 x 201 = 9.6k lattice cells, a 40 MB
# logit tensor per sample: per-sample working sets far above the host caches,
# like the full-length samples, whose 201k cells take ~15 min each on one
# core). Throughput is converted to the config's samples/s by lattice cells
# (the reference's cost is linear in cells: output-layer loops are 98 % of it,
# SURVEY §8(a)).
REF_T_SAMPLE = 48


def ref_sample_inputs(R, n, cfg_name):
    B, T, U, V, H = CONFIGS[cfg_name]
    t_full, u_full = R.padded_lengths(B, T, U)  # the reference's own ramp
    mean_cells = float(np.mean(t_full * (u_full + 1)))
    T_s = min(T, REF_T_SAMPLE)
    inp = R.synth_inputs(n, T_s, U, H, V)
    inp["t_len"][:] = T_s  # every sample at (T_s, U): equal work per worker
    inp["u_len"][:] = U
    rng = np.random.default_rng(1)
    inp["labels"][:] = rng.integers(1, V, inp["labels"].shape, dtype=np.int32)
    for k in ("acoustic", "label"):
        inp[k] = np.ascontiguousarray(inp[k])
    cells = float(np.sum(inp["t_len"] * (inp["u_len"] + 1)))
    return inp, mean_cells, cells, T_s


def run_reference(args, cfg_name):
    """The reference's own CPU engine (oracle/_ref: swt::run_step<float>,
    sample_wise_pr_dp, compiled unmodified from /root/reference) on a bounded
    sample of the workload with all the host threads it can use (the
    reference caps a DP group at 16, engine.cpp:336-352; budget 2^33 so
    Eq. 9 gives PI = 16 >= workers)."""
    from oracle import ref as R
    B, T, U, V, H = CONFIGS[cfg_name]
    if not R.available():
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref/libswt_ref.so not built"}))
        return
    cores = os.cpu_count() or 1
    workers = max(1, min(cores, 16))
    inp, mean_cells, cells, T_s = ref_sample_inputs(R, workers, cfg_name)
    run = lambda: R.run_step(inp, dtype=np.float32, mode="sample_wise_pr_dp",
                             budget=1 << 33, max_parallel=16, workers=workers)
    for _ in range(args.warmup):
        run()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
    step = float(np.median(times))
    value = (cells / mean_cells) / step
    sample = (f"{workers} samples of (T={T_s}, U={U}, V={V}, H={H}) per step "
              f"({cells:.0f} lattice cells), sample_wise_pr_dp, budget 2^33 (PI=16), "
              f"{workers} worker threads, run_step<float>; samples/s = cells/s / "
              f"{cfg_name}'s mean {mean_cells:.0f} cells/sample (padding ramp); "
              f"host: {cores} cores, {cpu_model()}")
    line = {"metric": METRIC, "value": value, "unit": "samples/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": step * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (reference synth_inputs, seed 1)",
            "config": {"workload": cfg_name, "B": B, "T": T, "U": U, "V": V,
                       "H": H, "H_A": H, "H_L": H, "engine": "swt::run_step (CPU)",
                       "deviation": f"bounded sample: {workers} samples of T={T_s} frames "
                                    f"(full U, V, H) per step, converted by lattice cells"},
            "cpu_baseline": {"value": value, "unit": "samples/s", "cores": workers,
                             "kind": "reference", "sample": sample},
            "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline_single(cfg_name):
    """Reference CPU engine, 1 thread, one bounded sample (rank 0, N=1)."""
    try:
        from oracle import ref as R
        if not R.available():
            return None
        inp, mean_cells, cells, T_s = ref_sample_inputs(R, 2, cfg_name)
        B, T, U, V, H = CONFIGS[cfg_name]
        t0 = time.perf_counter()
        R.run_step(inp, dtype=np.float32, mode="sample_wise_pr")
        dt = time.perf_counter() - t0
        return {"value": (cells / mean_cells) / dt, "unit": "samples/s",
                "cores": 1, "kind": "reference",
                "sample": f"2 samples (T={T_s}, U={U}, V={V}, H={H}; {cells:.0f} cells), "
                          f"run_step<float> sample_wise_pr, 1 thread, {dt:.1f} s; "
                          f"samples/s = cells/s / {cfg_name}'s mean {mean_cells:.0f} "
                          f"cells/sample; host {cpu_model()}"}
    except Exception as e:  # never let the baseline kill the GPU number
        return {"value": None, "unit": "samples/s", "cores": 1, "kind": "reference",
                "sample": f"failed: {e}"}


# ---------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=list(CONFIGS))
    ap.add_argument("--precision", default="fp16", choices=["fp16", "bf16", "bf16x", "tf32"])
    ap.add_argument("--group-cells", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-pageable", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            run_reference(args, args.config)
        return

    import torch
    import paper_2211_16270_b200 as sw

    dist = None
    # test hook (one-GPU boxes): every rank on GPU 0, gloo for the harness,
    # shard-only engines (no NCCL: one communicator cannot hold a GPU twice);
    # exercises the multi-rank orchestration, not the all-reduce
    shared = world > 1 and os.environ.get("SWTB_BENCH_SHARED_GPU") == "1"
    if world > 1:
        import torch.distributed as dist
        if shared:
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = local if world > 1 and not shared else 0
    torch.cuda.set_device(dev)

    B, T, U, V, H = CONFIGS[args.config]
    prec = sw.Precision[args.precision]

    nccl_id = None
    if world > 1 and not shared:
        obj = [sw.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    eng = sw.Engine(dev, prec, rank=rank, nranks=world, nccl_id=nccl_id,
                    group_cells=args.group_cells)

    batch, jp, op = sw.synth_inputs(B, T, U, H, V)
    cfg = sw.EngineConfig(mode=sw.EngineMode.sample_wise_pr_dp)
    stream = torch.cuda.ExternalStream(eng.stream, device=dev)

    # ---- device-resident inputs (value) ----
    # under torchrun each rank holds only its samples b % N == rank
    # (shard-local layout): per-GPU memory falls with N
    own = list(range(rank, B, world))
    shard_local = world > 1
    shard = (lambda x: np.ascontiguousarray(x[own])) if shard_local else (lambda x: x)
    B_rows = len(own) if shard_local else B
    d = lambda x: torch.from_numpy(x).to(f"cuda:{dev}")
    dbatch = sw.Batch(d(shard(batch.acoustic)), d(shard(batch.label)), d(shard(batch.labels)),
                      batch.t_len, batch.u_len, shard_local=shard_local)
    djp = sw.JointParams(d(jp.w_acoustic), d(jp.w_label), d(jp.bias))
    dop = sw.OutputParams(d(op.w_out), d(op.bias_out))
    z = lambda *s: torch.empty(*s, dtype=torch.float32, device=f"cuda:{dev}")
    dout = sw.GradientSet(z(H, H), z(H, H), z(H), z(V, H), z(V), z(B_rows, T, H),
                          z(B_rows, U + 1, H))
    dsl = z(B)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if shared else f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        r = eng.run_step(dbatch, djp, dop, cfg, out=dout, sample_losses=dsl)
    eng.reset_peak()
    torch.cuda.reset_peak_memory_stats(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier()
    # the timed region: K steps, no per-launch instrumentation (the stage
    # events cost ~2 % of the step; they run in a second pass below)
    with Clocks(dev) as clk:
        torch.cuda.nvtx.range_push("timed")  # ncu --nvtx-include timed/
        e0.record(stream)
        for _ in range(args.steps):
            r = eng.run_step(dbatch, djp, dop, cfg, out=dout, sample_losses=dsl)
        e1.record(stream)
        barrier()
        torch.cuda.nvtx.range_pop()
    ms_total = max_over_ranks(e0.elapsed_time(e1))
    ms_step = ms_total / args.steps
    value = B / (ms_step / 1e3)
    # per-kernel-kind device time (CUDA events around every launch, on the
    # engine's streams) over K more steps of the same workload: the
    # roofline's launch durations and the stage breakdown
    eng.set_profiling(True)
    eng.profile(reset=True)
    for _ in range(args.steps):
        eng.run_step(dbatch, djp, dop, cfg, out=dout, sample_losses=dsl)
    torch.cuda.synchronize(dev)
    eng.set_profiling(False)
    prof = eng.profile(reset=True)
    stats = r.stats
    loss = r.loss
    # device-resident path only (the e2e run below adds host-staging buffers)
    eng_peak = eng.peak_bytes()
    api_peak = torch.cuda.max_memory_allocated(dev)
    peak_gb = max_over_ranks((eng_peak + api_peak) / 1e9)

    # ---- e2e: pinned host buffers through the same C ABI call ----
    e2e = None
    if not args.no_e2e:
        pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()
        hbatch = sw.Batch(pin(shard(batch.acoustic)), pin(shard(batch.label)),
                          pin(shard(batch.labels)), batch.t_len, batch.u_len,
                          shard_local=shard_local)
        hjp = sw.JointParams(pin(jp.w_acoustic), pin(jp.w_label), pin(jp.bias))
        hop = sw.OutputParams(pin(op.w_out), pin(op.bias_out))
        hz = lambda *s: torch.empty(*s, dtype=torch.float32).pin_memory().numpy()
        hout = sw.GradientSet(hz(H, H), hz(H, H), hz(H), hz(V, H), hz(V),
                              hz(B_rows, T, H), hz(B_rows, U + 1, H))
        hsl = np.empty(B, np.float32)
        r2 = eng.run_step(hbatch, hjp, hop, cfg, out=hout, sample_losses=hsl)
        barrier()
        with Clocks(dev) as clk_e2e:
            t0 = time.perf_counter()
            for _ in range(args.steps):
                r2 = eng.run_step(hbatch, hjp, hop, cfg, out=hout, sample_losses=hsl)
            barrier()
            e2e_s = max_over_ranks(time.perf_counter() - t0) / args.steps
        e2e = {"value": B / e2e_s, "unit": "samples/s",
               "h2d_bytes_per_step": int(r2.stats["h2d_bytes"]),
               "d2h_bytes_per_step": int(r2.stats["d2h_bytes"]),
               "ms_per_step": e2e_s * 1e3,
               "loss_matches_device_path": bool(abs(r2.loss - loss) <= 1e-5 * abs(loss)),
               "clocks": clk_e2e.summary(), "host_buffers": "pinned"}
        # the same call with PAGEABLE host buffers (a drop-in caller's plain
        # std::vector tensors; the copies then go through driver staging)
        if not args.no_pageable:
            pg = lambda x: np.array(x, copy=True)
            pbatch = sw.Batch(pg(shard(batch.acoustic)), pg(shard(batch.label)),
                              pg(shard(batch.labels)), batch.t_len, batch.u_len,
                              shard_local=shard_local)
            pjp = sw.JointParams(pg(jp.w_acoustic), pg(jp.w_label), pg(jp.bias))
            pop = sw.OutputParams(pg(op.w_out), pg(op.bias_out))
            pz = lambda *s: np.zeros(s, np.float32)
            pout = sw.GradientSet(pz(H, H), pz(H, H), pz(H), pz(V, H), pz(V),
                                  pz(B_rows, T, H), pz(B_rows, U + 1, H))
            eng.run_step(pbatch, pjp, pop, cfg, out=pout, sample_losses=hsl)
            barrier()
            t0 = time.perf_counter()
            for _ in range(args.steps):
                eng.run_step(pbatch, pjp, pop, cfg, out=pout, sample_losses=hsl)
            barrier()
            pg_s = max_over_ranks(time.perf_counter() - t0) / args.steps
            e2e["pageable"] = {"value": B / pg_s, "unit": "samples/s", "ms_per_step": pg_s * 1e3,
                               "host_buffers": "pageable (numpy)"}
            del pbatch, pout

    # ---- secondary figure: plain bf16 operands (outside the north-star
    # fp32/TF32 bound: its own stated bound, tests/test_gpu_step.py) ----
    secondary = None
    if not args.no_secondary:
        eng.close()
        secondary = {}

        def timed_engine(precision, env=None):
            """samples/s of another engine configuration on the same inputs"""
            old = {k: os.environ.get(k) for k in (env or {})}
            os.environ.update(env or {})  # engine knobs are read at context creation
            try:
                nid = None
                if world > 1 and not shared:
                    obj = [sw.nccl_unique_id() if rank == 0 else None]
                    dist.broadcast_object_list(obj, src=0)
                    nid = obj[0]
                e2 = sw.Engine(dev, precision, rank=rank, nranks=world, nccl_id=nid,
                               group_cells=args.group_cells)
            finally:
                for k, v in old.items():
                    if v is None:
                        os.environ.pop(k, None)
                    else:
                        os.environ[k] = v
            s2 = torch.cuda.ExternalStream(e2.stream, device=dev)
            for _ in range(args.warmup):
                e2.run_step(dbatch, djp, dop, cfg, out=dout, sample_losses=dsl)
            barrier()
            f0 = torch.cuda.Event(enable_timing=True)
            f1 = torch.cuda.Event(enable_timing=True)
            f0.record(s2)
            for _ in range(args.steps):
                e2.run_step(dbatch, djp, dop, cfg, out=dout, sample_losses=dsl)
            f1.record(s2)
            barrier()
            ms2 = max_over_ranks(f0.elapsed_time(f1)) / args.steps
            e2.close()
            return {"value": B / (ms2 / 1e3), "unit": "samples/s", "ms_per_step": ms2}

        if prec == sw.Precision.fp16 and stats.get("active_tiles", -1) >= 0:
            # the same step with every tile in the backward (no zero-tile skip)
            secondary["fp16_dense_backward"] = timed_engine(
                sw.Precision.fp16, {"SWTB_SKIP_ZERO_TILES": "0"})
        if prec != sw.Precision.bf16:
            secondary["bf16"] = timed_engine(sw.Precision.bf16)
            secondary["bf16"]["parity_bound"] = "loss 5e-4, gradients 3e-2 (not the fp32 bound)"

    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---- roofline of the output-layer GEMM family (this rank's shard) ----
    burst, sustained, hbm, src = peaks()
    shard = list(range(rank, B, world))
    f_out, f_joint = algorithmic_flops(batch.t_len, batch.u_len, V, H, H, H, shard)
    # the GEMMs of the output layer: f^O forward, dz, dW_O, and the logit
    # recompute when dh is not formed from the stored logits (x slab; then
    # out_dh is an elementwise HBM pass on the lattice stream, not a GEMM)
    stored = bool(stats.get("logits_stored"))
    # zero-tile skip (fp16): the backward GEMMs walk only the active tiles;
    # their algorithmic work is 4 H V flops per cell of those tiles (the
    # skipped tiles' dh is exactly zero), the forward's 2 H V per cell
    active = int(stats.get("active_tiles", -1))
    active_frac = (active / max(1, int(stats["tiles"]))) if active >= 0 else 1.0
    f_dense = f_out
    f_out = f_out * (1.0 + 2.0 * active_frac) / 3.0
    fam = ("out_fwd", "out_dz", "out_dw") if stored else ("out_fwd", "out_dh", "out_dz", "out_dw")
    gemm_ms = sum(prof[k][0] for k in fam) / args.steps
    gemm_launches = sum(prof[k][1] for k in fam) // args.steps
    achieved = f_out / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else None
    peak = sustained if sustained else burst  # kernels timed inside a long step
    if prec == sw.Precision.tf32:
        peak = peak / 2
    f_all_out, f_all_joint = algorithmic_flops(batch.t_len, batch.u_len, V, H, H, H)
    f_all_total = f_all_out * (1.0 + 2.0 * active_frac) / 3.0 + f_all_joint
    kernels = {k: {"ms_per_step": v[0] / args.steps, "launches_per_step": v[1] // args.steps}
               for k, v in prof.items()}
    # DRAM traffic of the GEMM family: achieved DRAM GB/s of each GEMM kind in
    # the committed ncu --set full capture (profiles/), times its live
    # duration in this run (per step, the same basis as `achieved`)
    traffic, traffic_src = None, None
    tfile = TRAFFIC_STORED if stored else TRAFFIC_RECOMPUTE
    try:
        if tfile is None:
            raise FileNotFoundError
        with open(os.path.join(ROOT, "profiles", tfile)) as f:
            tj = json.load(f)
        kmap = {"out_fwd": "EpiFwdLse", "out_dh": "EpiBwdDh", "out_dz": "EpiDzGate", "out_dw": "EpiAtomic"}
        traffic = sum(tj["kernels"][kmap[k]]["achieved_dram_GBps"] * 1e9 * kernels[k]["ms_per_step"] / 1e3
                      for k in fam)
        traffic_src = (f"bytes/step: ncu dram__bytes_read+write rate per GEMM kind "
                       f"(profiles/{tfile}) x live duration")
    except Exception:
        pass
    # every libswt_b200 kernel launch of the last step (engine counter), x K
    launches = int(stats["kernel_launches"]) * args.steps

    cpu = None if (args.no_cpu_baseline or world > 1) else cpu_baseline_single(args.config)

    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": args.precision,
        "data": "synthetic (reference synth_inputs, seed 1, padding ramp)",
        "config": {"workload": args.config, "B": B, "T": T, "U": U, "V": V, "H": H,
                   "H_A": H, "H_L": H, "engine": "sample_wise_pr_dp (libswt_b200)",
                   "parallelism": f"sample-sharded dp{world}",
                   "l2": "inputs (h^A 2.1 GB at c4) exceed the 126 MB L2; no explicit flush",
                   "group_cells": args.group_cells or 1 << 20,
                   "output_gemm_precision": args.precision,
                   "zero_tile_skip": active >= 0,
                   "loss": loss},
        "peak_gb_per_gpu": peak_gb,
        "memory_model": memory_model(B, T, U, V, H, H, H, batch.t_len, batch.u_len),
        "peak_gb_breakdown": {"engine_workspace_gb": eng_peak / 1e9,
                              "api_tensors_gb": api_peak / 1e9},
        "roofline": {"bound": "tensor", "achieved": achieved,
                     "peak": peak, "unit": "TFLOP/s",
                     "frac": (achieved / peak) if achieved else None,
                     "traffic": traffic,
                     "traffic_source": traffic_src,
                     "kernel": "output-layer GEMM family (f^O fwd" + (", dz, dW_O; dh from the stored logits)" if stored else ", recompute+dh, dz, dW_O)"),
                     "per_kernel_executed_tflops": {
                         k: (f_dense / 3 * (1.0 if k == "out_fwd" else active_frac))
                         / (kernels[k]["ms_per_step"] / 1e3) / 1e12
                         for k in fam if kernels[k]["ms_per_step"] > 0},
                     "algorithmic_flops_per_step": f_out,
                     "algorithmic_flops_note": "2 H V per lattice cell (f^O forward) + 4 H V per "
                                               "cell of the tiles the backward walks (dz, dW_O); the "
                                               "logit recompute is executed, not credited",
                     "active_tile_fraction": active_frac,
                     "dense_equivalent_tflops": f_dense / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else None,
                     "launches_per_step": gemm_launches,
                     "duration_source": "CUDA events around every GEMM launch on the engine "
                                        "stream, K steps of the same workload right after "
                                        "the (uninstrumented) timed region",
                     "peak_source": f"{src} bf16 dense {'sustained' if sustained else 'burst'}"
                                    + (" / 2 for tf32" if prec == sw.Precision.tf32 else "")},
        "whole_step_tflops": f_all_total / (ms_step / 1e3) / 1e12 / world,
        "whole_step_dense_equivalent_tflops": (f_all_out + f_all_joint) / (ms_step / 1e3) / 1e12 / world,
        "kernels": kernels,
        "clocks": clk.summary(),
        "gpu_launches": launches,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "secondary": secondary,
        "stats": stats,
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
