"""TEST INFRASTRUCTURE ONLY — ctypes access to the unmodified reference
engine compiled from /root/reference/proj/core/src into
oracle/_ref/libswt_ref.so (see oracle/Makefile and oracle/ref_shim.cpp).

`available()` is False when the library was not built (e.g. a checkout
without /root/reference); callers then fall back to oracle.swt_oracle and
say so.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(_HERE, "_ref", "libswt_ref.so")
ACCEPTANCE = os.path.join(_HERE, "_ref", "acceptance")
REF_ROOT = "/root/reference/proj"

_lib = None


def build() -> bool:
    """Compile the reference (only possible where /root/reference exists)."""
    if not os.path.isdir(REF_ROOT):
        return os.path.exists(SO)
    subprocess.run(["make", "-C", _HERE, "ref"], check=True,
                   stdout=subprocess.DEVNULL)
    return True


def available() -> bool:
    return os.path.exists(SO)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{SO} not built")
        _lib = C.CDLL(SO)
        P = C.c_void_p
        I = C.c_int64
        _lib.ref_last_error.restype = C.c_char_p
        _lib.ref_synth_inputs.argtypes = [I] * 7 + [C.c_uint64] + [P] * 10
        for name in ("ref_run_step_f32", "ref_run_step_f64"):
            getattr(_lib, name).argtypes = ([I] * 7 + [P] * 10 +
                                            [C.c_int, I, C.c_int, C.c_int] +
                                            [P] * 9)
        _lib.ref_transducer_loss_f64.argtypes = [P, I, I, I, P, P, P]
        _lib.ref_enumerate_paths_loss.argtypes = [P, I, I, I, P, P]
        _lib.ref_count_paths.argtypes = [I, I]
        _lib.ref_count_paths.restype = I
        _lib.ref_parallel_iterations.argtypes = [I] * 4
        _lib.ref_padded_lengths.argtypes = [I, I, I, P, P]
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def _chk(rc):
    if rc != 0:
        raise RuntimeError(f"reference error {rc}: "
                           f"{lib().ref_last_error().decode()}")


def synth_inputs(B, T, U, H, V, H_A=None, H_L=None, seed=1) -> dict:
    H_A = H if H_A is None else H_A
    H_L = H if H_L is None else H_L
    f = lambda *s: np.empty(s, dtype=np.float32)
    d = dict(acoustic=f(B, T, H_A), label=f(B, U + 1, H_L),
             labels=np.empty((B, U), np.int32), t_len=np.empty(B, np.int64),
             u_len=np.empty(B, np.int64), w_acoustic=f(H, H_A),
             w_label=f(H, H_L), bias=f(H), w_out=f(V, H), bias_out=f(V))
    _chk(lib().ref_synth_inputs(B, T, U, H, H_A, H_L, V, seed,
                                *(_p(d[k]) for k in (
                                    "acoustic", "label", "labels", "t_len",
                                    "u_len", "w_acoustic", "w_label", "bias",
                                    "w_out", "bias_out"))))
    return d


MODES = {"batched": 0, "sample_wise": 1, "sample_wise_pr": 2,
         "sample_wise_pr_dp": 3}


def run_step(inp: dict, dtype=np.float64, mode="sample_wise_pr",
             budget=1_000_000_000, max_parallel=16, workers=1) -> dict:
    """swt::run_step<T> on `inp` (float32 inputs widened exactly for f64)."""
    g = lambda k: np.ascontiguousarray(inp[k], dtype=dtype)
    ac, lb = g("acoustic"), g("label")
    B, T, HA = ac.shape
    U1, HL = lb.shape[1], lb.shape[2]
    U = U1 - 1
    wa, wl, bz, wo, bo = (g(k) for k in ("w_acoustic", "w_label", "bias",
                                         "w_out", "bias_out"))
    H, V = wa.shape[0], wo.shape[0]
    labels = np.ascontiguousarray(inp["labels"], dtype=np.int32)
    t_len = np.ascontiguousarray(inp["t_len"], dtype=np.int64)
    u_len = np.ascontiguousarray(inp["u_len"], dtype=np.int64)
    z = lambda *s: np.zeros(s, dtype=dtype)
    out = dict(loss=z(1), sample_losses=z(B), dw_acoustic=z(H, HA),
               dw_label=z(H, HL), dbias=z(H), dw_out=z(V, H), dbias_out=z(V),
               dacoustic=z(B, T, HA), dlabel=z(B, U1, HL))
    fn = lib().ref_run_step_f64 if dtype == np.float64 else lib().ref_run_step_f32
    _chk(fn(B, T, U, HA, HL, H, V, _p(ac), _p(lb), _p(labels), _p(t_len),
            _p(u_len), _p(wa), _p(wl), _p(bz), _p(wo), _p(bo), MODES[mode],
            budget, max_parallel, workers,
            *(_p(out[k]) for k in ("loss", "sample_losses", "dw_acoustic",
                                   "dw_label", "dbias", "dw_out", "dbias_out",
                                   "dacoustic", "dlabel"))))
    out["loss"] = float(out["loss"][0])
    return out


def transducer_loss_sample(scores, y):
    scores = np.ascontiguousarray(scores, dtype=np.float64)
    T, U1, V = scores.shape
    yy = np.ascontiguousarray(y, dtype=np.int32)
    loss = np.zeros(1)
    ds = np.empty_like(scores)
    _chk(lib().ref_transducer_loss_f64(_p(scores), T, U1 - 1, V,
                                       _p(yy) if yy.size else None,
                                       _p(loss), _p(ds)))
    return float(loss[0]), ds


def enumerate_paths_loss(scores, y) -> float:
    scores = np.ascontiguousarray(scores, dtype=np.float64)
    T, U1, V = scores.shape
    yy = np.ascontiguousarray(y, dtype=np.int32)
    loss = np.zeros(1)
    _chk(lib().ref_enumerate_paths_loss(_p(scores), T, U1 - 1, V,
                                        _p(yy) if yy.size else None, _p(loss)))
    return float(loss[0])


def parallel_iterations(f, l, v, b) -> int:
    return int(lib().ref_parallel_iterations(f, l, v, b))


def padded_lengths(B, T, U):
    """swt::padded_lengths (reference bench.cpp:48-64)."""
    t = np.empty(B, np.int64)
    u = np.empty(B, np.int64)
    _chk(lib().ref_padded_lengths(B, T, U, _p(t), _p(u)))
    return t, u
