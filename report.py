#!/usr/bin/env python
"""Benchmark reports in the reference's schema.

Mirrors `swt bench` / `swt sweep` of the reference CLI
(proj/tools/swt_main.cpp:141-236) and its report format
(proj/core/src/bench.cpp:249-298: CSV columns
`mode,B,T,U,H,H_A,H_L,V,precision,median_step_seconds,peak_bytes,status,seed`,
JSON adds `loss_checksum`), with the step run by libswt_b200 on the GPU
(device-resident inputs from the reference generator `synth_inputs`).
`precision` is the reference's scalar-type field: "f32" (the inputs,
outputs and accumulators are float32, so the reference's parse_report_json,
bench.cpp:300-326, reads it back as f32); the JSON form adds
`operand_precision`, the output-layer GEMM operand type (fp16 / tf32 /
bf16x / bf16); `peak_bytes` is the engine's device high-water mark plus the API tensors;
`status` is "oom" when the device allocation fails (reference
OutOfMemoryError).

  python report.py bench --batch 8 --frames 64 --labels 16 --joint 128 --vocab 256
  python report.py sweep --axis batch --values 1,2,4,8 [...] --format json
  python report.py sweep --axis lengths --values 50x10,232x46,500x100 [...]
  python report.py sweep --axis lengths --values 100,200,400 [...]  # bare T: U scaled
  python report.py sweep --mode batched --axis batch --values 8,16,32 \
      --frames 1000 --labels 200 --joint 512 --vocab 1024   # batched comparator
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

COLUMNS = ("mode", "B", "T", "U", "H", "H_A", "H_L", "V", "precision",
           "median_step_seconds", "peak_bytes", "status", "seed")


def format_double(v: float) -> str:
    return "%.17g" % v  # reference format_double (bench.cpp:242-246)


class InvalidInputError(ValueError):
    """Mirrors swt::InvalidInputError (the reference CLI's exit code 2)."""


def parse_sweep_values(base, axis: str, values: str):
    """Reference parse_sweep_values (bench.cpp:171-221): comma-separated
    points; axis "batch": B values; axis "lengths": "TxU", or a bare T whose
    U is scaled by T / base T (rounded half away from zero, at least 1).
    Every value >= 1, at least one point, strictly ascending (B, or T)."""
    B0, T0, U0 = base
    points = []
    for item in values.split(","):
        if not item:
            continue
        try:
            if axis == "batch":
                p = (int(item), T0, U0)
            elif "x" in item:
                t, u = item.split("x", 1)
                p = (B0, int(t), int(u))
            else:  # bare T: U scales with T (std::llround)
                t = int(item)
                x = U0 * t / T0
                p = (B0, t, max(1, int(x + 0.5) if x >= 0 else -int(-x + 0.5)))
        except ValueError:
            raise InvalidInputError(f"cannot parse sweep value '{item}'") from None
        if min(p) < 1:
            raise InvalidInputError(f"sweep value '{item}' out of range")
        points.append(p)
    if not points:
        raise InvalidInputError("sweep needs at least one value")
    key = 0 if axis == "batch" else 1
    for a, b in zip(points, points[1:]):
        if not b[key] > a[key]:
            raise InvalidInputError("sweep values must ascend")
    return points


def emit(results, fmt: str) -> str:
    """Reference emit_report (bench.cpp:270-298)."""
    if not results:
        raise ValueError("refusing to emit an empty report")
    if fmt == "csv":
        out = ",".join(COLUMNS) + "\n"
        for r in results:
            out += ",".join(format_double(r[c]) if c == "median_step_seconds" else str(r[c])
                            for c in COLUMNS) + "\n"
        return out
    extra = ("loss_checksum", "operand_precision")
    return json.dumps([{**{c: r[c] for c in COLUMNS}, **{k: r[k] for k in extra if k in r}}
                       for r in results], indent=2) + "\n"


def run_point(B, T, U, H, HA, HL, V, mode, precision, warmup, steps, seed, ceiling=0):
    import torch
    import paper_2211_16270_b200 as sw
    res = {"mode": mode, "B": B, "T": T, "U": U, "H": H, "H_A": HA, "H_L": HL,
           "V": V, "precision": "f32", "operand_precision": precision, "seed": seed,
           "median_step_seconds": 0.0, "peak_bytes": 0, "status": "ok",
           "loss_checksum": 0.0}
    eng = sw.Engine(0, sw.Precision[precision])
    eng.set_alloc_ceiling(ceiling)  # reference --alloc-ceiling (0 = off)
    try:
        batch, jp, op = sw.synth_inputs(B, T, U, H, V, H_A=HA, H_L=HL, seed=seed)
        d = lambda x: torch.from_numpy(x).cuda()
        db = sw.Batch(d(batch.acoustic), d(batch.label), d(batch.labels), batch.t_len, batch.u_len)
        djp = sw.JointParams(d(jp.w_acoustic), d(jp.w_label), d(jp.bias))
        dop = sw.OutputParams(d(op.w_out), d(op.bias_out))
        cfg = sw.EngineConfig(mode=sw.EngineMode[mode])
        for _ in range(warmup):
            r = eng.run_step(db, djp, dop, cfg)
        eng.reset_peak()
        torch.cuda.reset_peak_memory_stats()
        times = []
        for _ in range(steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = eng.run_step(db, djp, dop, cfg)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
        res["median_step_seconds"] = statistics.median(times)
        res["peak_bytes"] = int(eng.peak_bytes() + torch.cuda.max_memory_allocated())
        res["loss_checksum"] = float(r.loss)
    except sw.OutOfMemoryError as e:  # reference bench.cpp:153-159
        res["status"] = "oom"
        res["oom_tensor"], res["oom_bytes"] = e.tensor, e.request_bytes
        res["peak_bytes"] = int(eng.peak_bytes())
    finally:
        eng.close()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("command", choices=["bench", "sweep"])
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--frames", type=int, default=64)
    ap.add_argument("--labels", type=int, default=16)
    ap.add_argument("--joint", type=int, default=128)
    ap.add_argument("--acoustic", type=int, default=0)
    ap.add_argument("--label-dim", type=int, default=0)
    ap.add_argument("--vocab", type=int, default=256)
    ap.add_argument("--mode", default="sample_wise_pr_dp",
                    choices=["batched", "sample_wise", "sample_wise_pr", "sample_wise_pr_dp"])
    ap.add_argument("--precision", default="fp16", choices=["fp16", "tf32", "bf16x", "bf16"])
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--alloc-ceiling", type=int, default=0,
                    help="simulated allocation ceiling in bytes (0 = off)")
    ap.add_argument("--axis", choices=["batch", "lengths"], default="batch")
    ap.add_argument("--values", default="")
    ap.add_argument("--format", choices=["csv", "json"], default="csv")
    a = ap.parse_args()
    HA = a.acoustic or a.joint
    HL = a.label_dim or a.joint
    points = [(a.batch, a.frames, a.labels)]
    if a.command == "sweep":
        try:
            points = parse_sweep_values((a.batch, a.frames, a.labels), a.axis, a.values)
        except InvalidInputError as e:  # reference CLI: exit code 2
            sys.stderr.write(f"error: {e}\n")
            sys.exit(2)
    results = [run_point(B, T, U, a.joint, HA, HL, a.vocab, a.mode, a.precision,
                         a.warmup, a.steps, a.seed, a.alloc_ceiling) for B, T, U in points]
    sys.stdout.write(emit(results, a.format))


if __name__ == "__main__":
    main()
