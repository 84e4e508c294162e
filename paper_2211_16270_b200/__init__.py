"""B200-native sample-wise transducer loss + gradients (arXiv 2211.16270).

Python mirror of the reference C++ engine API (``swt::run_step`` and
friends, reference proj/core/include/swt/engine.hpp) over the C ABI of
``libswt_b200.so`` (include/swt_b200.h). Host arrays are numpy; device arrays
may be any object exposing ``data_ptr()`` (e.g. torch CUDA tensors) — torch is
only plumbing here, every computation runs in libswt_b200's CUDA kernels.

There is no CPU fallback: if the shared library is missing this module fails
to import, and creating an Engine without an sm_100 GPU raises CudaError.
"""

from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import Any, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SWTB_LIB") or os.path.join(_HERE, "libswt_b200.so")

if not os.path.exists(LIB_PATH):  # fail loudly: no fallback path exists
    raise ImportError(
        f"{LIB_PATH} is missing; build it with `make -C {_HERE}` "
        "(or __graft_entry__.build())")

_lib = C.CDLL(LIB_PATH)


# ---------------------------------------------------------------------------
# C ABI declarations (include/swt_b200.h)

class _Opts(C.Structure):
    _fields_ = [("device", C.c_int), ("rank", C.c_int), ("nranks", C.c_int),
                ("nccl_id", C.c_void_p), ("precision", C.c_int),
                ("group_cells", C.c_int64)]


class _Batch(C.Structure):
    _fields_ = [("B", C.c_int64), ("T", C.c_int64), ("U", C.c_int64),
                ("H_A", C.c_int64), ("H_L", C.c_int64),
                ("acoustic", C.c_void_p), ("label", C.c_void_p),
                ("labels", C.c_void_p), ("t_len", C.c_void_p),
                ("u_len", C.c_void_p), ("location", C.c_int),
                ("shard_local", C.c_int), ("sample_weights", C.c_void_p)]


class _Params(C.Structure):
    _fields_ = [("H", C.c_int64), ("V", C.c_int64),
                ("w_acoustic", C.c_void_p), ("w_label", C.c_void_p),
                ("bias", C.c_void_p), ("w_out", C.c_void_p),
                ("bias_out", C.c_void_p), ("location", C.c_int)]


class _Cfg(C.Structure):
    _fields_ = [("mode", C.c_int), ("mem_budget_bytes", C.c_int64),
                ("max_parallel", C.c_int), ("worker_count", C.c_int),
                ("literal_pi_extents", C.c_int)]


class _Out(C.Structure):
    _fields_ = [("loss", C.c_void_p), ("sample_losses", C.c_void_p),
                ("dw_acoustic", C.c_void_p), ("dw_label", C.c_void_p),
                ("dbias", C.c_void_p), ("dw_out", C.c_void_p),
                ("dbias_out", C.c_void_p), ("dacoustic", C.c_void_p),
                ("dlabel", C.c_void_p), ("location", C.c_int)]


class _Stats(C.Structure):
    _fields_ = [("groups", C.c_int64), ("cells", C.c_int64),
                ("tiles", C.c_int64), ("kernel_launches", C.c_int64),
                ("parallel_iterations", C.c_int), ("peak_bytes", C.c_int64),
                ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64),
                ("logits_stored", C.c_int64), ("active_tiles", C.c_int64)]


class _SynthCfg(C.Structure):
    _fields_ = [("B", C.c_int64), ("T", C.c_int64), ("U", C.c_int64),
                ("H", C.c_int64), ("H_A", C.c_int64), ("H_L", C.c_int64),
                ("V", C.c_int64), ("seed", C.c_uint64)]


_P = C.c_void_p
_lib.swtb_abi_version.restype = C.c_int
_lib.swtb_ctx_create.argtypes = [C.POINTER(_Opts), C.POINTER(_P)]
_lib.swtb_ctx_create.restype = C.c_int
_lib.swtb_ctx_destroy.argtypes = [_P]
_lib.swtb_last_error.argtypes = [_P]
_lib.swtb_last_error.restype = C.c_char_p
_lib.swtb_stream.argtypes = [_P]
_lib.swtb_stream.restype = _P
_lib.swtb_set_caller_stream.argtypes = [_P, _P, C.c_int]
_lib.swtb_set_caller_stream.restype = C.c_int
_lib.swtb_step.argtypes = [_P, C.POINTER(_Batch), C.POINTER(_Params),
                           C.POINTER(_Cfg), C.POINTER(_Out)]
_lib.swtb_step.restype = C.c_int
_lib.swtb_get_stats.argtypes = [_P, C.POINTER(_Stats)]
_lib.swtb_get_stats.restype = C.c_int
_lib.swtb_peak_bytes.argtypes = [_P]
_lib.swtb_peak_bytes.restype = C.c_int64
_lib.swtb_reset_peak.argtypes = [_P]
_lib.swtb_set_alloc_ceiling.argtypes = [_P, C.c_int64]
_lib.swtb_set_deterministic.argtypes = [_P, C.c_int]
_lib.swtb_last_oom.argtypes = [_P, C.POINTER(C.c_int64), C.c_char_p, C.c_int64]
_lib.swtb_last_oom.restype = C.c_int
_lib.swtb_transducer_loss.argtypes = [_P, _P, C.c_int64, C.c_int64,
                                      C.c_int64, _P, _P, _P]
_lib.swtb_transducer_loss.restype = C.c_int
_lib.swtb_parallel_iterations.argtypes = [C.c_int64] * 4
_lib.swtb_parallel_iterations.restype = C.c_int
_lib.swtb_padded_lengths.argtypes = [C.c_int64, C.c_int64, C.c_int64, _P, _P]
_lib.swtb_padded_lengths.restype = C.c_int
_lib.swtb_synth_inputs.argtypes = [C.POINTER(_SynthCfg)] + [_P] * 10
_lib.swtb_synth_inputs.restype = C.c_int
_lib.swtb_debug_gemm.argtypes = [_P, C.c_int, C.c_int, C.c_int, _P, C.c_int64,
                                 _P, C.c_int64, C.c_int64, C.c_int64,
                                 C.c_int64, _P, C.c_int64, C.c_int]
_lib.swtb_debug_gemm.restype = C.c_int
_lib.swtb_set_profiling.argtypes = [_P, C.c_int]
_lib.swtb_get_profile.argtypes = [_P, _P, _P, C.c_int]
_lib.swtb_get_profile.restype = C.c_int
_lib.swtb_nccl_unique_id.argtypes = [_P]
_lib.swtb_nccl_unique_id.restype = C.c_int

#: swtb_stage names, index = enum value
STAGES = ("prep", "joint_fwd", "out_fwd", "lattice", "out_dh", "out_dz",
          "out_dw", "joint_bwd", "comm", "wait", "other")

#: every symbol include/swt_b200.h declares (checked by the CPU ABI test)
ABI_SYMBOLS = (
    "swtb_abi_version", "swtb_ctx_create", "swtb_ctx_destroy",
    "swtb_last_error", "swtb_stream", "swtb_step", "swtb_get_stats",
    "swtb_peak_bytes", "swtb_reset_peak", "swtb_transducer_loss",
    "swtb_parallel_iterations", "swtb_padded_lengths", "swtb_synth_inputs",
    "swtb_debug_gemm", "swtb_set_profiling", "swtb_get_profile",
    "swtb_nccl_unique_id", "swtb_set_alloc_ceiling", "swtb_last_oom",
    "swtb_set_deterministic", "swtb_set_caller_stream",
)


# ---------------------------------------------------------------------------
# Errors — the reference's swt::Error hierarchy (errors.hpp:12-66)

class SwtError(RuntimeError):
    """Base class (swt::Error)."""


class InvalidShapeError(SwtError):
    pass


class InvalidInputError(SwtError):
    pass


class NumericalDegeneracyError(SwtError):
    pass


class OutOfMemoryError(SwtError):
    """swt::OutOfMemoryError: ``tensor`` / ``request_bytes`` name the refused
    allocation (errors.hpp:37-53) when the engine reports them."""
    tensor: str = ""
    request_bytes: int = 0


class CudaError(SwtError):
    pass


class NcclError(SwtError):
    pass


_STATUS = {1: InvalidShapeError, 2: InvalidInputError,
           3: NumericalDegeneracyError, 4: OutOfMemoryError, 5: CudaError,
           6: NcclError, 7: SwtError}


def _check(status: int, ctx=None) -> None:
    if status != 0:
        msg = _lib.swtb_last_error(ctx).decode(errors="replace")
        err = _STATUS.get(status, SwtError)(msg)
        if status == 4 and ctx:
            nbytes, name = C.c_int64(0), C.create_string_buffer(64)
            if _lib.swtb_last_oom(ctx, C.byref(nbytes), name, 64) == 0:
                err.tensor, err.request_bytes = name.value.decode(), int(nbytes.value)
        raise err


# ---------------------------------------------------------------------------
# Reference-shaped types

class EngineMode(enum.IntEnum):
    """swt::EngineMode (engine.hpp:16-21)."""
    batched = 0
    sample_wise = 1
    sample_wise_pr = 2
    sample_wise_pr_dp = 3


class Precision(enum.IntEnum):
    """Output-layer GEMM operand precision (swtb_precision). fp16 and tf32
    meet the fp32 parity bound (loss 1e-4, gradients 1e-3); fp16 runs at the
    16-bit MMA rate."""
    bf16 = 0
    tf32 = 1
    bf16x = 2
    fp16 = 3


@dataclass
class EngineConfig:
    """swt::EngineConfig (engine.hpp:74-82)."""
    mode: EngineMode = EngineMode.sample_wise
    mem_budget_bytes: int = 1_000_000_000
    max_parallel: int = 16
    worker_count: int = 1
    literal_pi_extents: bool = False


@dataclass
class Batch:
    """swt::Batch<float> (engine.hpp:28-46). Arrays are numpy (host) or
    CUDA tensors (device); lengths are always host int64 arrays."""
    acoustic: Any   # [B, T, H_A] float32  (shard_local: [B_own, T, H_A])
    label: Any      # [B, U+1, H_L] float32
    labels: Any     # [B, U] int32, zero-padded
    t_len: np.ndarray  # [B] (always the whole batch)
    u_len: np.ndarray  # [B]
    # per-sample tensors (and dacoustic / dlabel outputs) hold only this
    # rank's samples b % nranks == rank, ascending (swtb_batch.shard_local)
    shard_local: bool = False
    # optional per-sample loss weights [B] >= 0 (host): gradients of
    # sum_b w_b L_b; losses stay unweighted (swtb_batch.sample_weights)
    sample_weights: Any = None

    @property
    def batch_size(self) -> int:
        return int(len(self.t_len))


@dataclass
class JointParams:
    """swt::JointParams (compute.hpp:13-23)."""
    w_acoustic: Any  # [H, H_A]
    w_label: Any     # [H, H_L]
    bias: Any        # [H]


@dataclass
class OutputParams:
    """swt::OutputParams (compute.hpp:25-32)."""
    w_out: Any     # [V, H]
    bias_out: Any  # [V]


@dataclass
class GradientSet:
    """swt::GradientSet (engine.hpp:49-58)."""
    dw_acoustic: Any
    dw_label: Any
    dbias: Any
    dw_out: Any
    dbias_out: Any
    dacoustic: Any
    dlabel: Any


@dataclass
class StepResult:
    """swt::StepResult (engine.hpp:84-89)."""
    loss: float
    sample_losses: Any
    grads: GradientSet
    stats: dict = field(default_factory=dict)


def _is_device(x) -> bool:
    return hasattr(x, "data_ptr") and getattr(x, "is_cuda", False)


def _ptr(x) -> int:
    if x is None:
        return 0
    if hasattr(x, "data_ptr"):
        return int(x.data_ptr())
    assert isinstance(x, np.ndarray) and x.flags.c_contiguous, \
        "host arrays must be C-contiguous numpy arrays"
    return int(x.ctypes.data)


def _f32(x):
    if hasattr(x, "data_ptr"):
        return x.contiguous()
    return np.ascontiguousarray(x, dtype=np.float32)


class Engine:
    """A libswt_b200 context on one GPU (optionally one rank of a
    multi-GPU sample-sharded job)."""

    def __init__(self, device: int = 0, precision: Precision = Precision.fp16,
                 rank: int = 0, nranks: int = 1,
                 nccl_id: Optional[bytes] = None, group_cells: int = 0):
        opts = _Opts(device, rank, nranks, None, int(precision), group_cells)
        self._nccl_buf = None
        if nccl_id is not None:  # None: shard-only (no collective); nranks=1: 1-rank comm
            _prefer_host_nccl()
            assert len(nccl_id) == 128
            self._nccl_buf = C.create_string_buffer(bytes(nccl_id), 128)
            opts.nccl_id = C.cast(self._nccl_buf, C.c_void_p)
        h = _P()
        _check(_lib.swtb_ctx_create(C.byref(opts), C.byref(h)))
        self._h = h
        self.device, self.precision = device, Precision(precision)
        self.rank, self.nranks = rank, nranks

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.swtb_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return int(_lib.swtb_stream(self._h) or 0)

    def stats(self) -> dict:
        s = _Stats()
        _check(_lib.swtb_get_stats(self._h, C.byref(s)), self._h)
        return {k: getattr(s, k) for k, _ in _Stats._fields_}

    def set_profiling(self, on: bool) -> None:
        _lib.swtb_set_profiling(self._h, int(bool(on)))

    def profile(self, reset: bool = False) -> dict:
        ms = (C.c_double * len(STAGES))()
        n = (C.c_int64 * len(STAGES))()
        _check(_lib.swtb_get_profile(self._h, ms, n, int(reset)), self._h)
        return {k: (ms[i], n[i]) for i, k in enumerate(STAGES)}

    def peak_bytes(self) -> int:
        return int(_lib.swtb_peak_bytes(self._h))

    def reset_peak(self) -> None:
        _lib.swtb_reset_peak(self._h)

    def set_deterministic(self, on: bool) -> None:
        """Bitwise-reproducible theta-grads (default on): ordered split-K
        reductions instead of fp32 atomics."""
        _lib.swtb_set_deterministic(self._h, int(bool(on)))

    def set_alloc_ceiling(self, nbytes: int) -> None:
        """Simulated device-memory ceiling (reference
        AllocationTracker::set_ceiling / BenchConfig.alloc_ceiling_bytes);
        0 turns it off."""
        _lib.swtb_set_alloc_ceiling(self._h, int(nbytes))

    # -- swt::run_step -------------------------------------------------------
    def run_step(self, batch: Batch, jp: JointParams, op: OutputParams,
                 cfg: EngineConfig = EngineConfig(),
                 out: Optional[GradientSet] = None,
                 sample_losses=None) -> StepResult:
        dev_in = _is_device(batch.acoustic)
        dev_par = _is_device(jp.w_acoustic)
        local = bool(getattr(batch, "shard_local", False))
        B_rows, T, HA = (int(s) for s in batch.acoustic.shape)
        B = len(batch.t_len) if local else B_rows
        B_own = (B - self.rank + self.nranks - 1) // self.nranks if self.rank < B else 0
        if local and B_rows != B_own:
            raise InvalidShapeError("shard-local batch must hold this rank's samples only")
        U1, HL = int(batch.label.shape[1]), int(batch.label.shape[2])
        U = U1 - 1
        H, V = int(op.w_out.shape[1]), int(op.w_out.shape[0])
        if tuple(batch.label.shape[:1]) != (B_rows,) or tuple(jp.w_acoustic.shape) != (H, HA) \
                or tuple(jp.w_label.shape) != (H, HL) or tuple(jp.bias.shape) != (H,) \
                or tuple(op.bias_out.shape) != (V,):
            raise InvalidShapeError("parameter extents do not match the batch")
        t_len = np.ascontiguousarray(batch.t_len, dtype=np.int64)
        u_len = np.ascontiguousarray(batch.u_len, dtype=np.int64)
        if t_len.shape != (B,) or u_len.shape != (B,):
            raise InvalidShapeError("batch length/label arrays are inconsistent")
        acoustic, label = _f32(batch.acoustic), _f32(batch.label)
        labels = batch.labels
        if not hasattr(labels, "data_ptr"):
            labels = np.ascontiguousarray(labels, dtype=np.int32)
        if tuple(labels.shape) != (B_rows, U) and U > 0:
            raise InvalidShapeError("batch length/label arrays are inconsistent")
        params = [_f32(x) for x in (jp.w_acoustic, jp.w_label, jp.bias,
                                    op.w_out, op.bias_out)]
        weights = getattr(batch, "sample_weights", None)
        if weights is not None:
            if hasattr(weights, "cpu"):
                weights = weights.detach().cpu().numpy()
            weights = np.ascontiguousarray(weights, dtype=np.float32)
            if weights.shape != (B,):
                raise InvalidShapeError("sample_weights must have one entry per sample")
        cb = _Batch(B, T, U, HA, HL, _ptr(acoustic), _ptr(label), _ptr(labels),
                    _ptr(t_len), _ptr(u_len), 1 if dev_in else 0, int(local),
                    _ptr(weights) if weights is not None else None)
        cp = _Params(H, V, *(_ptr(p) for p in params), 1 if dev_par else 0)
        cc = _Cfg(int(cfg.mode), int(cfg.mem_budget_bytes),
                  int(cfg.max_parallel), int(cfg.worker_count),
                  int(bool(cfg.literal_pi_extents)))
        if out is None:
            if dev_in:
                import torch
                dv = acoustic.device
                z = lambda *s: torch.empty(*s, dtype=torch.float32, device=dv)
            else:
                z = lambda *s: np.empty(s, dtype=np.float32)
            out = GradientSet(z(H, HA), z(H, HL), z(H), z(V, H), z(V),
                              z(B_rows, T, HA), z(B_rows, U1, HL))
        dev_out = _is_device(out.dw_out)
        if sample_losses is None:
            if dev_out:
                import torch
                sample_losses = torch.empty(B, dtype=torch.float32,
                                            device=out.dw_out.device)
            else:
                sample_losses = np.empty(B, dtype=np.float32)
            sl_ptr, dev_sl = _ptr(sample_losses), dev_out
        else:
            sl_ptr, dev_sl = _ptr(sample_losses), _is_device(sample_losses)
        if dev_sl != dev_out:
            raise InvalidInputError("sample_losses must live with the outputs")
        loss = np.zeros(1, dtype=np.float32)
        loss_dev = None
        if dev_out:
            import torch
            loss_dev = torch.zeros(1, dtype=torch.float32, device=out.dw_out.device)
        co = _Out(_ptr(loss_dev) if dev_out else _ptr(loss), sl_ptr,
                  *(_ptr(g) for g in (out.dw_acoustic, out.dw_label, out.dbias,
                                      out.dw_out, out.dbias_out,
                                      out.dacoustic, out.dlabel)),
                  1 if dev_out else 0)
        if dev_in or dev_par or dev_out:
            # device tensors may still be being written by torch's current
            # stream: the step's stream waits on it (swtb_set_caller_stream)
            import torch
            cs = torch.cuda.current_stream(self.device).cuda_stream
            _check(_lib.swtb_set_caller_stream(self._h, cs or None, 1), self._h)
        _check(_lib.swtb_step(self._h, C.byref(cb), C.byref(cp), C.byref(cc),
                              C.byref(co)), self._h)
        total = float(loss_dev.item()) if dev_out else float(loss[0])
        return StepResult(total, sample_losses, out, self.stats())

    # -- testing hook: one core GEMM on device tensors ----------------------
    def debug_gemm(self, A, B, out, *, a_mn=False, b_mn=False,
                   precision=Precision.bf16, accumulate=False):
        M = A.shape[1] if a_mn else A.shape[0]
        K = A.shape[0] if a_mn else A.shape[1]
        N = B.shape[1] if b_mn else B.shape[0]
        _check(_lib.swtb_debug_gemm(self._h, int(precision), int(a_mn),
                                    int(b_mn), _ptr(A), A.stride(0), _ptr(B),
                                    B.stride(0), M, N, K, _ptr(out),
                                    out.stride(0), int(accumulate)), self._h)

    # -- swt::transducer_loss_sample (f^W on explicit scores) ----------------
    def transducer_loss_sample(self, scores: np.ndarray, labels):
        scores = np.ascontiguousarray(scores, dtype=np.float64)
        if scores.ndim != 3:
            raise InvalidShapeError("scores must be [frames, labels+1, vocab]")
        T, U1, V = scores.shape
        y = np.ascontiguousarray(np.asarray(labels, dtype=np.int32).reshape(-1))
        if y.shape[0] != U1 - 1:
            raise InvalidInputError(
                f"label count {y.shape[0]} does not match lattice label rows {U1}")
        loss = np.zeros(1, dtype=np.float64)
        ds = np.empty_like(scores)
        _check(_lib.swtb_transducer_loss(self._h, _ptr(scores), T, U1 - 1, V,
                                         _ptr(y) if y.size else None,
                                         _ptr(loss), _ptr(ds)), self._h)
        return float(loss[0]), ds


# ---------------------------------------------------------------------------
# Context-free helpers

def _prefer_host_nccl() -> None:
    """Make the process's NCCL (torch's, when present) the one libswt_b200
    binds to, before it resolves NCCL on first multi-GPU use."""
    try:
        import torch  # noqa: F401  (loads its bundled libnccl.so.2)
    except Exception:
        pass


def nccl_unique_id() -> bytes:
    _prefer_host_nccl()
    buf = C.create_string_buffer(128)
    _check(_lib.swtb_nccl_unique_id(buf))
    return buf.raw


def abi_version() -> int:
    return int(_lib.swtb_abi_version())


def compute_parallel_iterations(frames: int, labels: int, vocab: int,
                                budget_bytes: int) -> int:
    """Eq. 9 (reference engine.cpp:31-50)."""
    r = _lib.swtb_parallel_iterations(frames, labels, vocab, budget_bytes)
    if r < 0:
        raise InvalidInputError(_lib.swtb_last_error(None).decode())
    return int(r)


def padded_lengths(batch: int, max_frames: int, max_labels: int):
    """Benchmark padding ramp (reference bench.cpp:48-64)."""
    t = np.empty(batch, dtype=np.int64)
    u = np.empty(batch, dtype=np.int64)
    _check(_lib.swtb_padded_lengths(batch, max_frames, max_labels,
                                    _ptr(t), _ptr(u)))
    return t, u


def synth_inputs(B: int, T: int, U: int, H: int, V: int, H_A: int = None,
                 H_L: int = None, seed: int = 1):
    """Bit-identical to swt::synth_inputs<float> (bench.cpp:66-115).
    Returns (Batch, JointParams, OutputParams) of host numpy arrays."""
    H_A = H if H_A is None else H_A
    H_L = H if H_L is None else H_L
    f = lambda *s: np.empty(s, dtype=np.float32)
    ac, lb = f(B, T, H_A), f(B, U + 1, H_L)
    labels = np.empty((B, U), dtype=np.int32)
    t_len, u_len = np.empty(B, np.int64), np.empty(B, np.int64)
    wa, wl, bz, wo, bo = f(H, H_A), f(H, H_L), f(H), f(V, H), f(V)
    cfg = _SynthCfg(B, T, U, H, H_A, H_L, V, seed)
    _check(_lib.swtb_synth_inputs(C.byref(cfg), *(_ptr(x) for x in (
        ac, lb, labels, t_len, u_len, wa, wl, bz, wo, bo))))
    return (Batch(ac, lb, labels, t_len, u_len), JointParams(wa, wl, bz),
            OutputParams(wo, bo))


def run_step(batch: Batch, jp: JointParams, op: OutputParams,
             cfg: EngineConfig = EngineConfig(), device: int = 0,
             precision: Precision = Precision.fp16) -> StepResult:
    """One-shot swt::run_step on `device` (creates and frees a context)."""
    eng = Engine(device, precision)
    try:
        return eng.run_step(batch, jp, op, cfg)
    finally:
        eng.close()
