#!/usr/bin/env python
"""CPU emulation of the output-layer operand roundings (test tooling, not the
product): which operand formats keep the step inside the north-star bound
(loss 1e-4 relative, gradients 1e-3 max-relative per tensor)?

Every GEMM of the output layer is emulated as float64 arithmetic on operands
rounded to the format the GPU kernel stages them in; accumulation error
(fp32 in TMEM) is ignored. Formats: f64 (exact), tf32 (cvt.rna), bf16 (RNE),
fp16 (RNE, optional power-of-two scale), and "<fmt>x" = hi + lo pair of that
format (two MMAs). Usage:

  python scripts/precision_study.py --cfg c3 --samples 0,127 \
      --plan z=fp16,wf=fp16x,dh=fp16s,wd=fp16x
"""

import argparse
import sys
import os

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from oracle import swt_oracle as O  # noqa: E402


def rnd(x, fmt):
    x = np.asarray(x, dtype=np.float64)
    if fmt in ("f64", None):
        return x
    if fmt.endswith("x"):
        base = fmt[:-1]
        hi = rnd(x, base)
        return hi + rnd(x - hi, base)
    if fmt == "f32":
        return x.astype(np.float32).astype(np.float64)
    x32 = x.astype(np.float32)
    if fmt == "bf16":
        u = x32.view(np.uint32).astype(np.uint64)
        u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
        return u.astype(np.uint32).view(np.float32).astype(np.float64)
    if fmt == "tf32":  # cvt.rna.tf32.f32: nearest, ties away
        u = x32.view(np.uint32).astype(np.uint64)
        u = (u + 0x1000) & 0xFFFFE000
        return u.astype(np.uint32).view(np.float32).astype(np.float64)
    if fmt == "fp16":
        return x32.astype(np.float16).astype(np.float64)
    if fmt == "fp16d":  # rounded twice: an fp16 softmax term, then the scaled product
        u = np.random.default_rng(7).uniform(0.5, 1.0, x32.shape)  # the per-block scale
        s16 = (x32 / u).astype(np.float16).astype(np.float64)
        return (s16 * u).astype(np.float32).astype(np.float16).astype(np.float64)
    if fmt.startswith("fp16s"):  # scaled by 2^k so the max maps near 2^14
        m = np.max(np.abs(x32)) if x32.size else 0.0
        k = 0 if m == 0 else 14 - int(np.floor(np.log2(m)))
        s = 2.0 ** k
        return (x32 * s).astype(np.float16).astype(np.float64) / s
    raise ValueError(fmt)


def tanh_approx(x):
    # tanh.approx.f32: max relative error ~2^-11; emulate as a worst-ish case
    t = np.tanh(x)
    return t * (1.0 + 2.0 ** -11 * np.sign(np.sin(1e4 * x)))


def process_sample(a, l, y, wa, wl, bz, wo, bo, P):
    pa = a @ wa.T
    pl = l @ wl.T
    pre = pa[:, None, :] + pl[None, :, :] + bz
    if P.get("tanh") == "f16x2":  # tanh.approx.f16x2 on fp16-rounded inputs
        x16 = pre.astype(np.float32).astype(np.float16).astype(np.float64)
        z = np.tanh(x16) * (1.0 + 2.0 ** -10.5 * np.sign(np.sin(1e4 * pre)))
    elif P.get("tanh") == "approx":
        z = tanh_approx(pre)
    else:
        z = np.tanh(pre)
    T, U1, H = z.shape
    V = wo.shape[0]
    zq = rnd(z.reshape(-1, H), P["z"])
    if P["wf"].endswith("m"):  # single rounding + mean-z correction of the logits
        whi = rnd(wo, P["wf"][:-1])
        dW = (wo - whi).T
        z3 = zq.reshape(T, U1, -1)
        if P.get("corr") == "tu":  # additive two-way fit z ~ zt + zu - zbar
            zt, zu, zb = z3.mean(axis=1), z3.mean(axis=0), zq.mean(axis=0)
            c = (zt @ dW)[:, None, :] + (zu @ dW)[None, :, :] - (zb @ dW)
        elif P.get("corr") == "u":
            c = ((z3.mean(axis=0)) @ dW)[None, :, :]
        elif P.get("corr", "").startswith("u"):  # mean over a frame subsample
            n = int(P["corr"][1:])
            ts = np.unique((np.arange(n) * T) // n)
            c = ((z3[ts].mean(axis=0)) @ dW)[None, :, :]
        else:
            c = (zq.mean(axis=0) @ dW)[None, None, :]
        scores = (zq @ whi.T).reshape(T, U1, V) + c + bo
    else:
        scores = (zq @ rnd(wo, P["wf"]).T + bo).reshape(T, U1, V)
    den = O.log_denominator(scores)
    alpha, beta = O.forward_backward(scores, den, y)
    loss = -beta[0, 0]
    if P.get("wr", P["wf"]) != P["wf"]:
        scores = (zq @ rnd(wo, P["wr"]).T + bo).reshape(T, U1, V)
    dh = O.loss_gradient(scores, den, alpha, beta, y)
    dhf = dh.reshape(-1, V)
    dhq = rnd(dhf, P["dh"])
    dz = (dhq @ rnd(wo, P["wd"])).reshape(T, U1, H)
    dwo = rnd(dhf, P.get("dhw", P["dh"])).T @ rnd(zq, P.get("zw", P["z"]))
    dbo = dhq.sum(axis=0)
    zg = zq.reshape(T, U1, H)
    g = dz * (1.0 - zg * zg)
    ga = g.sum(axis=1)
    gl = g.sum(axis=0)
    return (loss, ga.T @ a, gl.T @ l, ga.sum(axis=0), dwo, dbo, ga @ wa, gl @ wl)


def run(inp, samples, P):
    f = lambda k: np.asarray(inp[k], dtype=np.float64)
    ac, lb = f("acoustic"), f("label")
    wa, wl, bz, wo, bo = (f(k) for k in ("w_acoustic", "w_label", "bias", "w_out", "bias_out"))
    out = {k: 0.0 for k in ("loss",) + O.GRAD_KEYS}
    da, dl = [], []
    for b in samples:
        tb, ub = int(inp["t_len"][b]), int(inp["u_len"][b])
        r = process_sample(ac[b, :tb], lb[b, :ub + 1], inp["labels"][b, :ub], wa, wl, bz, wo, bo, P)
        out["loss"] += r[0]
        for k, v in zip(("dw_acoustic", "dw_label", "dbias", "dw_out", "dbias_out"), r[1:6]):
            out[k] = out[k] + v
        da.append(r[6])
        dl.append(r[7])
    out["dacoustic"] = np.concatenate(da)
    out["dlabel"] = np.concatenate(dl)
    return out


CFG = {"c2": (32, 200, 50, 512, 256), "c3": (128, 500, 100, 1024, 512),
       "c4": (1024, 1000, 200, 1024, 512), "c5": (256, 750, 150, 4096, 640)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="c3")
    ap.add_argument("--samples", default="0")
    ap.add_argument("--plan", action="append", required=True)
    a = ap.parse_args()
    B, T, U, V, H = CFG[a.cfg]
    inp = O.synth_inputs(B, T, U, H, V)
    samples = [int(s) for s in a.samples.split(",")]
    ref = run(inp, samples, dict(z="f64", wf="f64", dh="f64", wd="f64"))
    for plan in a.plan:
        P = dict(kv.split("=") for kv in plan.split(","))
        r = run(inp, samples, P)
        errs = {k: O.rel_err(r[k], ref[k]) for k in O.GRAD_KEYS}
        le = abs(r["loss"] - ref["loss"]) / abs(ref["loss"])
        worst = max(errs, key=errs.get)
        print(f"{a.cfg} {samples} {plan:45s} loss {le:.1e}  worst {worst} {errs[worst]:.2e}  "
              + " ".join(f"{k[1:]}={v:.1e}" for k, v in errs.items()), flush=True)


if __name__ == "__main__":
    main()
