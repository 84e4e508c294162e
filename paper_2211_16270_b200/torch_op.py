"""Encoder hand-off (arXiv 2211.16270 Algorithm 1 lines 13-14; SURVEY §8(f)
row 3): the sample-wise transducer loss as a ``torch.autograd.Function``.

``transducer_loss(h_a, h_l, labels, t_len, u_len, w_a, w_l, b_z, w_o, b_o)``
returns the per-sample losses; its backward hands dh^A / dh^L straight to the
encoders' autograd graph as device tensors (no host copies) and fills the
joint / output parameters' gradients. The forward already computes every
gradient (that is the sample-wise method: logits are never kept). When the
incoming per-sample loss gradient g is the same for every sample (sum / mean
losses, the training case) backward only scales the cached gradients. For a
per-sample weighting, backward re-runs the step with those weights
(swtb_batch.sample_weights: the gradients of sum_b g_b L_b); negative
weights take two weighted steps (g+ and g-).

All arithmetic runs in libswt_b200 (C ABI) on the tensors' device; torch is
only the container. There is no CPU path.
"""

from __future__ import annotations

from typing import Dict, Optional

import numpy as np
import torch

from . import (Batch, Engine, EngineConfig, EngineMode, GradientSet,
               JointParams, OutputParams, Precision)

_engines: Dict[tuple, Engine] = {}


def _engine(device: torch.device, precision: Precision) -> Engine:
    key = (device.index or 0, int(precision))
    if key not in _engines:
        _engines[key] = Engine(device.index or 0, precision)
    return _engines[key]


class TransducerLoss(torch.autograd.Function):
    @staticmethod
    def _step(eng, h_a, h_l, labels, t_len, u_len, w_a, w_l, b_z, w_o, b_o, weights=None):
        f = lambda x: x.detach().float().contiguous()
        B, T, HA = h_a.shape
        U1, HL = h_l.shape[1], h_l.shape[2]
        H, V = w_o.shape[1], w_o.shape[0]
        z = lambda *s: torch.empty(*s, dtype=torch.float32, device=h_a.device)
        grads = GradientSet(z(H, HA), z(H, HL), z(H), z(V, H), z(V), z(B, T, HA), z(B, U1, HL))
        losses = z(B)
        lab = labels.detach().to(torch.int32).contiguous()
        r = eng.run_step(
            Batch(f(h_a), f(h_l), lab, np.asarray(t_len.cpu() if torch.is_tensor(t_len) else t_len, np.int64),
                  np.asarray(u_len.cpu() if torch.is_tensor(u_len) else u_len, np.int64),
                  sample_weights=weights),
            JointParams(f(w_a), f(w_l), f(b_z)), OutputParams(f(w_o), f(b_o)),
            EngineConfig(mode=EngineMode.sample_wise_pr_dp), out=grads, sample_losses=losses)
        return r, grads

    @staticmethod
    def forward(ctx, h_a, h_l, labels, t_len, u_len, w_a, w_l, b_z, w_o, b_o,
                precision=Precision.fp16, engine=None):
        if not h_a.is_cuda:
            raise RuntimeError("transducer_loss needs CUDA tensors (libswt_b200 has no CPU path)")
        eng = engine or _engine(h_a.device, Precision(precision))
        r, grads = TransducerLoss._step(eng, h_a, h_l, labels, t_len, u_len, w_a, w_l, b_z, w_o, b_o)
        ctx.save_for_backward(grads.dacoustic, grads.dlabel, grads.dw_acoustic,
                              grads.dw_label, grads.dbias, grads.dw_out, grads.dbias_out,
                              h_a, h_l, labels, w_a, w_l, b_z, w_o, b_o)
        ctx.lengths = (t_len, u_len)
        ctx.eng = eng
        ctx.dtypes = (h_a.dtype, h_l.dtype, w_a.dtype, w_l.dtype, b_z.dtype, w_o.dtype, b_o.dtype)
        return r.sample_losses

    @staticmethod
    def backward(ctx, g):
        dac, dlb, dwa, dwl, dbz, dwo, dbo, h_a, h_l, labels, w_a, w_l, b_z, w_o, b_o = \
            ctx.saved_tensors
        t = ctx.dtypes
        g = g.reshape(-1)
        if g.numel() <= 1 or bool(torch.all(g == g[0])):
            s = g[0]
            out = (dac.mul(s), dlb.mul(s), dwa.mul(s), dwl.mul(s), dbz.mul(s), dwo.mul(s),
                   dbo.mul(s))
        else:
            # per-sample weights: the gradients of sum_b g_b L_b, by one
            # weighted step (two when g has both signs: g+ minus g-)
            gw = g.detach().float().cpu().numpy()
            args = (h_a, h_l, labels) + ctx.lengths + (w_a, w_l, b_z, w_o, b_o)
            parts = []
            for sign, w in ((1.0, np.maximum(gw, 0.0)), (-1.0, np.maximum(-gw, 0.0))):
                if np.any(w > 0):
                    _, gr = TransducerLoss._step(ctx.eng, *args, weights=w)
                    parts.append((sign, gr))
            out = []
            for k in ("dacoustic", "dlabel", "dw_acoustic", "dw_label", "dbias", "dw_out",
                      "dbias_out"):
                acc = None
                for sign, gr in parts:
                    v = getattr(gr, k) * sign
                    acc = v if acc is None else acc + v
                out.append(acc)
        return (out[0].to(t[0]), out[1].to(t[1]), None, None, None,
                out[2].to(t[2]), out[3].to(t[3]), out[4].to(t[4]),
                out[5].to(t[5]), out[6].to(t[6]), None, None)


def transducer_loss(h_a, h_l, labels, t_len, u_len, w_a, w_l, b_z, w_o, b_o,
                    precision: Precision = Precision.fp16,
                    engine: Optional[Engine] = None) -> torch.Tensor:
    """Per-sample transducer losses [B] with libswt_b200 gradients attached."""
    return TransducerLoss.apply(h_a, h_l, labels, t_len, u_len, w_a, w_l, b_z,
                                w_o, b_o, precision, engine)
