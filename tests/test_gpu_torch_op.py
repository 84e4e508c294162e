"""GPU: the encoder hand-off — libswt_b200's step as a
torch.autograd.Function. dh^A / dh^L flow into upstream encoder layers as
device tensors; the joint/output parameter gradients land in .grad. Checked
against the float64 oracle through the chain rule (tf32 bound)."""

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_2211_16270_b200 as sw  # noqa: E402
from paper_2211_16270_b200.torch_op import transducer_loss  # noqa: E402
from oracle import swt_oracle as O  # noqa: E402


def test_autograd_handoff_matches_oracle():
    batch, jp, op = sw.synth_inputs(6, 40, 12, 48, 64, H_A=32, H_L=24, seed=3)
    dev = torch.device("cuda", 0)
    t = lambda x, g=True: torch.tensor(x, device=dev, requires_grad=g)
    # a tiny "encoder" in front of the loss: h_a = x_a @ P (so dP = x_a^T dh_a)
    rng = np.random.default_rng(0)
    x_a = rng.standard_normal(batch.acoustic.shape).astype(np.float32) * 0.1
    proj = np.eye(batch.acoustic.shape[2], dtype=np.float32)
    P = t(proj)
    h_a = torch.tensor(x_a, device=dev) @ P
    h_a_np = (x_a @ proj)
    for b in range(6):  # padded frames stay zero (the API contract)
        h_a_np[b, batch.t_len[b]:] = 0
    mask = torch.zeros_like(h_a)
    for b in range(6):
        mask[b, : batch.t_len[b]] = 1
    h_a = h_a * mask
    h_l = t(batch.label)
    params = [t(jp.w_acoustic), t(jp.w_label), t(jp.bias), t(op.w_out), t(op.bias_out)]
    losses = transducer_loss(h_a, h_l, torch.tensor(batch.labels, device=dev),
                             batch.t_len, batch.u_len, *params,
                             precision=sw.Precision.tf32)
    total = losses.sum()
    total.backward()

    inp = dict(acoustic=h_a_np, label=batch.label, labels=batch.labels, t_len=batch.t_len,
               u_len=batch.u_len, w_acoustic=jp.w_acoustic, w_label=jp.w_label,
               bias=jp.bias, w_out=op.w_out, bias_out=op.bias_out)
    ref = O.run_step(inp)
    assert abs(float(total) - ref["loss"]) <= 1e-4 * ref["loss"]
    for p, k in zip(params, ("dw_acoustic", "dw_label", "dbias", "dw_out", "dbias_out")):
        assert O.rel_err(p.grad.cpu().numpy(), ref[k]) < 1e-3, k
    assert O.rel_err(h_l.grad.cpu().numpy(), ref["dlabel"]) < 1e-3
    # chain rule into the encoder layer
    dP_ref = np.einsum("btk,btj->kj", x_a * mask.cpu().numpy(), ref["dacoustic"])
    assert O.rel_err(P.grad.cpu().numpy(), dP_ref) < 1e-3


def test_mean_reduction_scales_gradients():
    batch, jp, op = sw.synth_inputs(4, 30, 8, 32, 40, seed=9)
    dev = torch.device("cuda", 0)
    t = lambda x: torch.tensor(x, device=dev, requires_grad=True)
    a1, a2 = t(batch.acoustic), t(batch.acoustic)
    w1, w2 = t(op.w_out), t(op.w_out)
    common = lambda a, w: transducer_loss(
        a, torch.tensor(batch.label, device=dev), torch.tensor(batch.labels, device=dev),
        batch.t_len, batch.u_len, torch.tensor(jp.w_acoustic, device=dev),
        torch.tensor(jp.w_label, device=dev), torch.tensor(jp.bias, device=dev), w,
        torch.tensor(op.bias_out, device=dev), precision=sw.Precision.tf32)
    common(a1, w1).sum().backward()
    common(a2, w2).mean().backward()
    assert O.rel_err(a2.grad.cpu().numpy() * 4, a1.grad.cpu().numpy()) < 1e-6
    assert O.rel_err(w2.grad.cpu().numpy() * 4, w1.grad.cpu().numpy()) < 1e-6


@pytest.mark.parametrize("weights", [[0.5, 2.0, 0.0, 1.25], [1.0, -0.5, 2.0, 0.25]])
def test_per_sample_loss_weights(weights):
    """sum_b w_b L_b: backward re-runs the step with swtb_batch.sample_weights
    (two weighted steps when the weights have both signs); checked against
    the oracle's per-sample gradients combined with the same weights."""
    batch, jp, op = sw.synth_inputs(4, 30, 8, 32, 40, seed=9)
    dev = torch.device("cuda", 0)
    t = lambda x: torch.tensor(x, device=dev, requires_grad=True)
    a, l, wo = t(batch.acoustic), t(batch.label), t(op.w_out)
    losses = transducer_loss(a, l, torch.tensor(batch.labels, device=dev), batch.t_len,
                             batch.u_len, torch.tensor(jp.w_acoustic, device=dev),
                             torch.tensor(jp.w_label, device=dev),
                             torch.tensor(jp.bias, device=dev), wo,
                             torch.tensor(op.bias_out, device=dev), precision=sw.Precision.tf32)
    w = torch.tensor(weights, device=dev)
    (losses * w).sum().backward()
    inp = dict(acoustic=batch.acoustic, label=batch.label, labels=batch.labels,
               t_len=batch.t_len, u_len=batch.u_len, w_acoustic=jp.w_acoustic,
               w_label=jp.w_label, bias=jp.bias, w_out=op.w_out, bias_out=op.bias_out)
    ref_wo = 0.0
    ref_da = np.zeros(batch.acoustic.shape)
    ref_dl = np.zeros(batch.label.shape)
    for b, wb in enumerate(weights):
        r = O.run_step(inp, samples=[b])
        ref_wo = ref_wo + wb * r["dw_out"]
        ref_da[b] = wb * r["dacoustic"][b]
        ref_dl[b] = wb * r["dlabel"][b]
    assert O.rel_err(wo.grad.cpu().numpy(), ref_wo) < 1e-3
    assert O.rel_err(a.grad.cpu().numpy(), ref_da) < 1e-3
    assert O.rel_err(l.grad.cpu().numpy(), ref_dl) < 1e-3
    # the losses themselves are unweighted
    ref_l = [O.run_step(inp, samples=[b])["sample_losses"][b] for b in range(4)]
    assert np.allclose(losses.detach().cpu().numpy(), ref_l, rtol=1e-4)
