"""GPU: the four engine modes — the batched comparator
(reference run_batched, engine.cpp:245-323: whole batch at padded extents,
every intermediate materialized), the padded sample-wise engine and the +PR
engines give the same results; their device memory behaves like the
reference's (acceptance.cpp criteria 5, 6 and 8: sample-wise memory almost
independent of B, peak ordering, OOM simulation under an allocation
ceiling)."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2211_16270_b200 as sw  # noqa: E402
from oracle import swt_oracle as O  # noqa: E402

MODES = [sw.EngineMode.batched, sw.EngineMode.sample_wise,
         sw.EngineMode.sample_wise_pr, sw.EngineMode.sample_wise_pr_dp]
GRADS = ("dw_acoustic", "dw_label", "dbias", "dw_out", "dbias_out", "dacoustic", "dlabel")


def _ragged(seed=5):
    batch, jp, op = sw.synth_inputs(6, 41, 11, 48, 72, H_A=40, H_L=24, seed=seed)
    # non-monotone lengths, one U_b = 0 sample; padding re-zeroed
    batch.t_len[:] = [41, 3, 29, 17, 1, 36]
    batch.u_len[:] = [11, 0, 7, 11, 2, 5]
    for b in range(6):
        batch.acoustic[b, batch.t_len[b]:] = 0
        batch.label[b, batch.u_len[b] + 1:] = 0
        batch.labels[b, batch.u_len[b]:] = 0
        batch.labels[b, :batch.u_len[b]] = 1 + (np.arange(batch.u_len[b]) * 5 + b) % 71
    return batch, jp, op


def _oracle(batch, jp, op):
    return O.run_step(dict(acoustic=batch.acoustic, label=batch.label, labels=batch.labels,
                           t_len=batch.t_len, u_len=batch.u_len, w_acoustic=jp.w_acoustic,
                           w_label=jp.w_label, bias=jp.bias, w_out=op.w_out,
                           bias_out=op.bias_out))


@pytest.mark.parametrize("mode", MODES, ids=lambda m: m.name)
def test_every_mode_matches_oracle(mode):
    batch, jp, op = _ragged()
    ref = _oracle(batch, jp, op)
    eng = sw.Engine(0, sw.Precision.tf32)
    r = eng.run_step(batch, jp, op, sw.EngineConfig(mode=mode))
    assert abs(r.loss - ref["loss"]) <= 1e-4 * abs(ref["loss"])
    np.testing.assert_allclose(r.sample_losses, ref["sample_losses"], rtol=1e-4)
    for k in GRADS:
        assert O.rel_err(getattr(r.grads, k), ref[k]) < 1e-3, k
    # padded slots stay exactly zero in every mode
    for b in range(6):
        assert not r.grads.dacoustic[b, batch.t_len[b]:].any()
        assert not r.grads.dlabel[b, batch.u_len[b] + 1:].any()
    eng.close()


def test_four_modes_agree_on_50_random_ragged_batches():
    # acceptance.cpp criterion 3 (B <= 8, T <= 12, U <= 5), every mode against
    # the f64 oracle at the tf32 bound
    rng = np.random.default_rng(303)
    eng = sw.Engine(0, sw.Precision.tf32)
    for i in range(50):
        B, T, U = int(rng.integers(1, 9)), int(rng.integers(1, 13)), int(rng.integers(1, 6))
        H, V = int(rng.integers(4, 20)), int(rng.integers(2, 12))
        batch, jp, op = sw.synth_inputs(B, T, U, H, V, H_A=int(rng.integers(3, 12)),
                                        H_L=int(rng.integers(3, 12)), seed=1000 + i)
        batch.t_len[:] = rng.integers(1, T + 1, B)
        batch.u_len[:] = rng.integers(0, U + 1, B)
        for b in range(B):
            batch.acoustic[b, batch.t_len[b]:] = 0
            batch.label[b, batch.u_len[b] + 1:] = 0
            batch.labels[b, batch.u_len[b]:] = 0
            batch.labels[b, :batch.u_len[b]] = rng.integers(1, V, batch.u_len[b])
        ref = _oracle(batch, jp, op)
        for mode in MODES:
            r = eng.run_step(batch, jp, op, sw.EngineConfig(mode=mode))
            assert abs(r.loss - ref["loss"]) <= 1e-4 * abs(ref["loss"]), (i, mode)
            for k in GRADS:
                assert O.rel_err(getattr(r.grads, k), ref[k]) < 1e-3, (i, mode, k)
    eng.close()


def test_batched_equals_sample_wise_bf16():
    # reference test_bench.cpp:109-129: batched vs sample-wise loss checksum
    batch, jp, op = sw.synth_inputs(8, 50, 10, 64, 128, seed=1)
    eng = sw.Engine(0, sw.Precision.bf16)
    a = eng.run_step(batch, jp, op, sw.EngineConfig(mode=sw.EngineMode.batched))
    b = eng.run_step(batch, jp, op, sw.EngineConfig(mode=sw.EngineMode.sample_wise_pr_dp))
    assert abs(a.loss - b.loss) <= 1e-4 * abs(b.loss)
    for k in GRADS:
        assert O.rel_err(getattr(a.grads, k), getattr(b.grads, k)) < 2e-2, k
    eng.close()


def _trio_bytes(T, U1, H, V):  # reference lattice_trio_bytes (engine.cpp:52-55), f32
    return T * U1 * (H + 2 * V) * 4


def test_oom_simulation_fails_batched_only():
    # acceptance.cpp:415-447 (criterion 8): ceiling = half the analytic
    # batched 4D footprint at B=16, T=50, U=10, H=64, V=128
    B, T, U, H, V = 16, 50, 10, 64, 128
    batch, jp, op = sw.synth_inputs(B, T, U, H, V, seed=22)
    ceiling = B * _trio_bytes(T, U + 1, H, V) // 2
    eng = sw.Engine(0)
    eng.set_alloc_ceiling(ceiling)
    with pytest.raises(sw.OutOfMemoryError) as ei:
        eng.run_step(batch, jp, op, sw.EngineConfig(mode=sw.EngineMode.batched))
    assert ei.value.tensor and ei.value.request_bytes > 0
    assert "exceeds ceiling %d" % ceiling in str(ei.value)
    eng.close()
    losses = []
    for mode in MODES[1:]:
        e = sw.Engine(0)
        e.set_alloc_ceiling(ceiling)
        r = e.run_step(batch, jp, op, sw.EngineConfig(mode=mode))
        assert e.peak_bytes() <= ceiling
        losses.append(r.loss)
        e.close()
    assert max(losses) - min(losses) <= 1e-4 * abs(losses[0])


def _peak(mode, B, group_cells=0, prec=sw.Precision.bf16):
    batch, jp, op = sw.synth_inputs(B, 50, 10, 64, 128, seed=3)
    e = sw.Engine(0, prec, group_cells=group_cells)
    e.run_step(batch, jp, op, sw.EngineConfig(mode=mode))
    p = e.peak_bytes()
    e.close()
    return p


def test_peak_ordering():
    # acceptance criterion 6: peak(pr) <= peak(sample_wise) <= peak(batched)
    for B in (2, 4, 16):
        p_pr = _peak(sw.EngineMode.sample_wise_pr, B)
        p_sw = _peak(sw.EngineMode.sample_wise, B)
        p_b = _peak(sw.EngineMode.batched, B)
        assert p_pr <= p_sw <= p_b, (B, p_pr, p_sw, p_b)


def test_memory_scaling_with_batch_size():
    # acceptance criterion 5 (Fig. 2): one sample per group, the sample-wise
    # engine grows per added sample by its 3D tensors (h^A, h^L staged in,
    # dh^A, dh^L out; x1.2 covers the per-sample plan descriptors) once its
    # joint-network batch (SWTB_JOINT_BATCH groups, 8 by default) is full,
    # while the batched comparator grows by at least 0.8x its 4D tensors
    # (joint, scores, dscores at the padded, tile-rounded extents)
    T, U1, H, V = 50, 11, 64, 128
    jb = max(1, int(os.environ.get("SWTB_JOINT_BATCH", "8")))
    three_d = 2 * (T * H + U1 * H) * 4
    tiles = -(-T // 16) * -(-U1 // 8)
    four_d = tiles * 128 * (H * 2 + V * 4 + V * 2)  # bf16 operands, fp32 scores
    s0 = _peak(sw.EngineMode.sample_wise, jb, group_cells=T * U1)
    b4 = _peak(sw.EngineMode.batched, 4)
    for k in (4, 16):  # fixed per-step overheads amortised over 3-15 batches
        B = k * jb
        ps = _peak(sw.EngineMode.sample_wise, B, group_cells=T * U1)
        pb = _peak(sw.EngineMode.batched, B)
        assert ps - s0 <= 1.2 * (B - jb) * three_d, (B, ps - s0)
        assert pb - b4 >= 0.8 * (B - 4) * four_d, (B, pb - b4)


@pytest.mark.parametrize("mode", MODES, ids=lambda m: m.name)
def test_bitwise_determinism(mode):
    # acceptance criterion 10: fixed inputs give bitwise-identical runs, also
    # across contexts (split-K partials are reduced in a fixed order)
    for dims in ((7, 12, 5, 10, 12, 8, 8), (8, 120, 30, 256, 512, 256, 256)):
        B, T, U, H, V, HA, HL = dims
        batch, jp, op = sw.synth_inputs(B, T, U, H, V, H_A=HA, H_L=HL, seed=24)
        runs = []
        for _ in range(2):
            e = sw.Engine(0, sw.Precision.bf16)
            runs.append(e.run_step(batch, jp, op, sw.EngineConfig(mode=mode)))
            runs.append(e.run_step(batch, jp, op, sw.EngineConfig(mode=mode)))
            e.close()
        for r in runs[1:]:
            assert r.loss == runs[0].loss
            assert np.array_equal(r.sample_losses, runs[0].sample_losses)
            for k in GRADS:
                assert np.array_equal(getattr(r.grads, k), getattr(runs[0].grads, k)), (dims, k)
