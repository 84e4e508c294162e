"""TEST INFRASTRUCTURE ONLY — the CPU oracle for libswt_b200's parity tests.

Never imported by the product package (paper_2211_16270_b200/). Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / reference arm use it,
and only as the checker.

float64 restatement of the reference's sample-wise transducer step
(/root/reference/proj, paths below relative to it). Sequential pieces (RNG,
alpha/beta recursion, path enumeration) are plain C in swt_oracle.c; the
dense linear algebra is numpy (float64 BLAS). Pinned against the compiled
reference (oracle/_ref, see ref.py) and against its known-answer tests by
tests/test_oracle_cpu.py and tests/golden/.

  synth_inputs            core/src/bench.cpp:66-115, core/include/swt/rng.hpp
  joint_forward           core/src/compute.cpp:45-67
  output_forward          core/src/compute.cpp:69-90
  log_denominator         core/src/loss.cpp:31-39 (tensor.hpp:397-405)
  forward_backward        core/src/loss.cpp:41-81
  loss_gradient           core/src/loss.cpp:83-132
  output_backward         core/src/compute.cpp:92-122
  joint_backward          core/src/compute.cpp:124-192
  run_step (sample-wise)  core/src/engine.cpp:150-243, 325-398
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "liboracle.so")


def build() -> None:
    subprocess.run(["make", "-C", _HERE, "_build/liboracle.so"], check=True,
                   stdout=subprocess.DEVNULL)


if not os.path.exists(_SO):
    build()
_lib = C.CDLL(_SO)
_P = C.c_void_p
_lib.orc_synth_inputs.argtypes = [C.c_int64] * 7 + [C.c_uint64] + [_P] * 10
_lib.orc_synth_inputs.restype = C.c_int
_lib.orc_padded_lengths.argtypes = [C.c_int64] * 3 + [_P, _P]
_lib.orc_parallel_iter.argtypes = [C.c_int64] * 4
_lib.orc_parallel_iter.restype = C.c_int
_lib.orc_lattice.argtypes = [_P, _P, C.c_int64, C.c_int64, _P, _P]
_lib.orc_lattice.restype = C.c_double
_lib.orc_count_paths.argtypes = [C.c_int64, C.c_int64]
_lib.orc_count_paths.restype = C.c_int64
_lib.orc_enumerate_loss.argtypes = [_P, _P, C.c_int64, C.c_int64, C.c_int64]
_lib.orc_enumerate_loss.restype = C.c_double
_lib.orc_mt64_first.argtypes = [C.c_uint64, C.c_int64, _P]
_lib.orc_mt64_first.restype = C.c_uint64
_lib.orc_log_add_exp.argtypes = [C.c_double, C.c_double]
_lib.orc_log_add_exp.restype = C.c_double

BLANK = 0


def _p(a: np.ndarray) -> int:
    assert a.flags.c_contiguous
    return a.ctypes.data


class OracleInputError(ValueError):
    """Mirrors swt::InvalidInputError."""


class OracleDegeneracyError(ArithmeticError):
    """Mirrors swt::NumericalDegeneracyError."""


# ---------------------------------------------------------------------------
# measurement inputs

def mt19937_64(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.uint64)
    _lib.orc_mt64_first(seed, n, _p(out))
    return out


def padded_lengths(B: int, T: int, U: int):
    t = np.empty(B, np.int64)
    u = np.empty(B, np.int64)
    _lib.orc_padded_lengths(B, T, U, _p(t), _p(u))
    return t, u


def synth_inputs(B, T, U, H, V, H_A=None, H_L=None, seed=1) -> dict:
    H_A = H if H_A is None else H_A
    H_L = H if H_L is None else H_L
    f = lambda *s: np.empty(s, dtype=np.float32)
    d = dict(acoustic=f(B, T, H_A), label=f(B, U + 1, H_L),
             labels=np.empty((B, U), np.int32), t_len=np.empty(B, np.int64),
             u_len=np.empty(B, np.int64), w_acoustic=f(H, H_A),
             w_label=f(H, H_L), bias=f(H), w_out=f(V, H), bias_out=f(V))
    rc = _lib.orc_synth_inputs(
        B, T, U, H, H_A, H_L, V, seed,
        *(_p(d[k]) for k in ("acoustic", "label", "labels", "t_len", "u_len",
                             "w_acoustic", "w_label", "bias", "w_out",
                             "bias_out")))
    if rc:
        raise OracleInputError("all benchmark dimensions must be >= 1")
    return d


def compute_parallel_iterations(frames, labels, vocab, budget) -> int:
    r = _lib.orc_parallel_iter(frames, labels, vocab, budget)
    if r < 0:
        raise OracleInputError("parallel-iteration extents must be >= 1")
    return int(r)


def count_paths(frames: int, labels: int) -> int:
    return int(_lib.orc_count_paths(frames, labels))


# ---------------------------------------------------------------------------
# f^W (per-sample loss)

def log_denominator(scores: np.ndarray) -> np.ndarray:
    m = scores.max(axis=-1, keepdims=True)
    with np.errstate(invalid="ignore"):
        s = np.exp(scores - m).sum(axis=-1)
    out = m[..., 0] + np.log(s)
    return np.where(np.isneginf(m[..., 0]), -np.inf, out)


def _lp(scores, log_den, y):
    T, U1, V = scores.shape
    lpb = np.ascontiguousarray(scores[:, :, BLANK] - log_den, dtype=np.float64)
    lpy = np.zeros((T, U1), dtype=np.float64)
    if U1 > 1:
        yy = np.asarray(y, dtype=np.int64)
        lpy[:, :U1 - 1] = np.take_along_axis(
            scores[:, :U1 - 1, :], yy[None, :, None].repeat(T, 0), axis=2)[..., 0] \
            - log_den[:, :U1 - 1]
    return lpb, lpy


def _check_labels(y, U1, V):
    if len(y) != U1 - 1:
        raise OracleInputError("label count does not match lattice label rows")
    for l in y:
        if l <= BLANK or l >= V:
            raise OracleInputError(f"label id {l} outside [1, {V})")


def forward_backward(scores, log_den, y):
    T, U1, V = scores.shape
    if T < 1:
        raise OracleInputError("lattice needs at least one frame")
    _check_labels(y, U1, V)
    lpb, lpy = _lp(scores, log_den, y)
    alpha = np.empty((T, U1))
    beta = np.empty((T, U1))
    _lib.orc_lattice(_p(lpb), _p(lpy), T, U1, _p(alpha), _p(beta))
    return alpha, beta


def loss_gradient(scores, log_den, alpha, beta, y):
    T, U1, V = scores.shape
    log_z = beta[0, 0]
    if not np.isfinite(log_z):
        raise OracleDegeneracyError("total path log-probability is not finite")
    shift = alpha - log_den - log_z                       # [T, U1]
    g = scores + shift[..., None]
    d = np.exp(g + beta[..., None])
    bdest = np.full((T, U1), -np.inf)
    bdest[:-1, :] = beta[1:, :]
    bdest[-1, -1] = 0.0
    d[:, :, BLANK] -= np.exp(g[:, :, BLANK] + bdest)
    if U1 > 1:
        yy = np.asarray(y, dtype=np.int64)
        idx = yy[None, :, None].repeat(T, 0)
        gy = np.take_along_axis(g[:, :U1 - 1, :], idx, axis=2)[..., 0]
        sub = np.exp(gy + beta[:, 1:])
        tt, uu = np.meshgrid(np.arange(T), np.arange(U1 - 1), indexing="ij")
        d[tt, uu, yy[uu]] -= sub
    if not np.all(np.isfinite(d)):
        raise OracleDegeneracyError("non-finite output-score gradient")
    return d


def transducer_loss_sample(scores: np.ndarray, y):
    """(loss, dscores) — reference loss.cpp:176-185."""
    scores = np.asarray(scores, dtype=np.float64)
    den = log_denominator(scores)
    alpha, beta = forward_backward(scores, den, y)
    if not np.isfinite(beta[0, 0]):
        raise OracleDegeneracyError("no alignment path carries mass")
    return -beta[0, 0], loss_gradient(scores, den, alpha, beta, y)


def enumerate_paths_loss(scores, y, max_paths=1_000_000) -> float:
    scores = np.asarray(scores, dtype=np.float64)
    den = log_denominator(scores)
    lpb, lpy = _lp(scores, den, y)
    T, U1, _ = scores.shape
    r = _lib.orc_enumerate_loss(_p(lpb), _p(lpy), T, U1, max_paths)
    if r == -1e300:
        raise OverflowError("instance has too many paths")
    return float(r)


# ---------------------------------------------------------------------------
# full step

def process_sample(a, l, y, wa, wl, bz, wo, bo):
    """One cropped sample -> (loss, dwa, dwl, dbz, dwo, dbo, da, dl), f64.
    a [T_b, H_A], l [U_b+1, H_L] (engine.cpp:150-214 with PR)."""
    pa = a @ wa.T                                  # [T, H]
    pl = l @ wl.T                                  # [U1, H]
    z = np.tanh(pa[:, None, :] + pl[None, :, :] + bz)   # [T, U1, H]
    T, U1, H = z.shape
    V = wo.shape[0]
    zf = z.reshape(-1, H)
    scores = (zf @ wo.T + bo).reshape(T, U1, V)
    loss, dh = transducer_loss_sample(scores, y)
    dhf = dh.reshape(-1, V)
    dz = (dhf @ wo).reshape(T, U1, H)
    dwo = dhf.T @ zf
    dbo = dhf.sum(axis=0)
    g = dz * (1.0 - z * z)
    ga = g.sum(axis=1)                             # [T, H]
    gl = g.sum(axis=0)                             # [U1, H]
    return (loss, ga.T @ a, gl.T @ l, ga.sum(axis=0), dwo, dbo,
            ga @ wa, gl @ wl)


def run_step(inp: dict, samples=None) -> dict:
    """Sample-wise (+PR) step in float64 on `inp` (arrays as from
    synth_inputs; float32 inputs are widened exactly). `samples` restricts
    the step to a subset of batch indices (theta-grads summed over it)."""
    f = lambda k: np.asarray(inp[k], dtype=np.float64)
    ac, lb = f("acoustic"), f("label")
    wa, wl, bz, wo, bo = (f(k) for k in ("w_acoustic", "w_label", "bias",
                                         "w_out", "bias_out"))
    labels = np.asarray(inp["labels"], dtype=np.int64)
    t_len = np.asarray(inp["t_len"], dtype=np.int64)
    u_len = np.asarray(inp["u_len"], dtype=np.int64)
    B, T, HA = ac.shape
    U1, HL = lb.shape[1], lb.shape[2]
    H, V = wa.shape[0], wo.shape[0]
    out = dict(loss=0.0, sample_losses=np.zeros(B),
               dw_acoustic=np.zeros((H, HA)), dw_label=np.zeros((H, HL)),
               dbias=np.zeros(H), dw_out=np.zeros((V, H)), dbias_out=np.zeros(V),
               dacoustic=np.zeros((B, T, HA)), dlabel=np.zeros((B, U1, HL)))
    for b in (range(B) if samples is None else samples):
        tb, ub = int(t_len[b]), int(u_len[b])
        y = labels[b, :ub] if labels.ndim == 2 else labels[b * (U1 - 1):][:ub]
        r = process_sample(ac[b, :tb], lb[b, :ub + 1], y, wa, wl, bz, wo, bo)
        out["sample_losses"][b] = r[0]
        out["loss"] += r[0]
        out["dw_acoustic"] += r[1]
        out["dw_label"] += r[2]
        out["dbias"] += r[3]
        out["dw_out"] += r[4]
        out["dbias_out"] += r[5]
        out["dacoustic"][b, :tb] = r[6]
        out["dlabel"][b, :ub + 1] = r[7]
    return out


GRAD_KEYS = ("dw_acoustic", "dw_label", "dbias", "dw_out", "dbias_out",
             "dacoustic", "dlabel")


def rel_err(x, ref) -> float:
    """Per-tensor normalized error max|x - ref| / max|ref|."""
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    den = np.max(np.abs(ref))
    if den == 0:
        return float(np.max(np.abs(x)))
    return float(np.max(np.abs(x - ref)) / den)
