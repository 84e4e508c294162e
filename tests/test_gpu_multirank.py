"""GPU: the multi-GPU code paths of libswt_b200 on one device.

* the NCCL collective path: a real communicator (ncclCommInitRank, here with
  one rank) and the step's ncclAllReduce of the theta-grads + losses;
* shard-local layouts (swtb_batch.shard_local): a rank's per-sample tensors
  and its device staging hold only its samples (b % nranks == rank), so a
  rank's memory shrinks with the number of ranks;
* a rank that owns no sample (nranks > B);
* the caller-stream contract (swtb_set_caller_stream): inputs written
  asynchronously on a torch side stream are complete before the step reads
  them.
Reference: engine.cpp:359-396 (sample loop), 390-395 (ordered loss sum)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_2211_16270_b200 as sw  # noqa: E402
from oracle import swt_oracle as O  # noqa: E402

P = sw.Precision.fp16


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def grads(r):
    g = {k: getattr(r.grads, k) for k in O.GRAD_KEYS}
    g = {k: (v.cpu().numpy() if hasattr(v, "cpu") else np.asarray(v)) for k, v in g.items()}
    sl = r.sample_losses
    g["sample_losses"] = sl.cpu().numpy() if hasattr(sl, "cpu") else np.asarray(sl)
    return g


@pytest.fixture(scope="module")
def case():
    batch, jp, op = sw.synth_inputs(9, 80, 20, 96, 128, H_A=64, H_L=48, seed=5)
    e = sw.Engine(0, P)
    ref = grads(e.run_step(batch, jp, op))
    e.close()
    return batch, jp, op, ref


def test_single_rank_nccl_communicator_runs_the_allreduce(case):
    batch, jp, op, ref = case
    e = sw.Engine(0, P, rank=0, nranks=1, nccl_id=sw.nccl_unique_id())
    e.set_profiling(True)
    r = e.run_step(batch, jp, op)
    prof = e.profile(reset=True)
    e.close()
    assert prof["comm"][0] > 0.0  # the all-reduce ran inside the step
    g = grads(r)
    for k in O.GRAD_KEYS + ("sample_losses",):
        assert np.array_equal(g[k], ref[k]), k  # sum over one rank: exact


@pytest.mark.parametrize("host", [False, True])
def test_shard_local_layout_matches_full_layout(case, host):
    """Each of 3 shard-only ranks gets only its samples (device or host
    buffers); its dh^A / dh^L rows equal the full run's slots of those
    samples and the partial theta-grads sum to the full result."""
    batch, jp, op, ref = case
    B, nr = batch.batch_size, 3
    tot = {k: 0.0 for k in ("dw_acoustic", "dw_label", "dbias", "dw_out", "dbias_out",
                            "sample_losses")}
    peaks = []
    for rank in range(nr):
        own = list(range(rank, B, nr))
        cvt = (lambda x: np.ascontiguousarray(x)) if host else dev
        lb = sw.Batch(cvt(batch.acoustic[own]), cvt(batch.label[own]), cvt(batch.labels[own]),
                      batch.t_len, batch.u_len, shard_local=True)
        jpx = jp if host else sw.JointParams(dev(jp.w_acoustic), dev(jp.w_label), dev(jp.bias))
        opx = op if host else sw.OutputParams(dev(op.w_out), dev(op.bias_out))
        e = sw.Engine(0, P, rank=rank, nranks=nr)
        r = e.run_step(lb, jpx, opx)
        peaks.append(e.peak_bytes())
        e.close()
        g = grads(r)
        assert g["dacoustic"].shape[0] == len(own)
        assert O.rel_err(g["dacoustic"], ref["dacoustic"][own]) < 1e-5
        assert O.rel_err(g["dlabel"], ref["dlabel"][own]) < 1e-5
        for k in tot:
            tot[k] = tot[k] + g[k]
    for k in tot:
        assert O.rel_err(tot[k], ref[k]) < 2e-4, k


def test_host_staging_holds_only_the_rank_shard():
    """With host buffers a rank stages only its own samples on the device:
    at 4 ranks the engine's staging bytes fall ~4x."""
    batch, jp, op = sw.synth_inputs(32, 200, 40, 64, 64)

    def peak(rank, nr):
        e = sw.Engine(0, P, rank=rank, nranks=nr)
        e.run_step(batch, jp, op)
        p = e.peak_bytes()
        e.close()
        return p
    one, four = peak(0, 1), peak(0, 4)
    staging = 32 * (200 * 64 + 41 * 64) * 4 * 2  # inputs + dh outputs, all samples
    assert one - four > 0.6 * staging


def test_rank_without_samples():
    batch, jp, op = sw.synth_inputs(3, 20, 5, 32, 16)
    e = sw.Engine(0, P, rank=5, nranks=8)
    # host outputs: slots of samples a rank does not own are left untouched
    z = lambda *s: np.zeros(s, np.float32)
    out = sw.GradientSet(z(32, 32), z(32, 32), z(32), z(16, 32), z(16), z(3, 20, 32), z(3, 6, 32))
    r = e.run_step(batch, jp, op, out=out)
    e.close()
    g = grads(r)
    assert r.loss == 0.0
    for k in O.GRAD_KEYS + ("sample_losses",):
        assert not np.any(g[k]), k


def test_inputs_from_a_side_stream_are_ordered():
    """Inputs produced on a non-blocking torch stream right before the call:
    the step waits for that stream (swtb_set_caller_stream), no host sync."""
    batch, jp, op = sw.synth_inputs(4, 120, 30, 128, 256)
    e = sw.Engine(0, P)
    ref = grads(e.run_step(batch, jp, op))
    s = torch.cuda.Stream()
    src = [dev(x) for x in (batch.acoustic, batch.label, jp.w_acoustic, jp.w_label,
                            jp.bias, op.w_out, op.bias_out)]
    labels = dev(batch.labels)
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        big = torch.randn(4096, 4096, device="cuda")
        for _ in range(8):  # keep the side stream busy before the copies
            big = big @ big.T / 4096.0
        dst = [torch.empty_like(x) for x in src]
        for d, x in zip(dst, src):
            d.copy_(x + 0.0 * big[0, 0])
        r = e.run_step(sw.Batch(dst[0], dst[1], labels, batch.t_len, batch.u_len),
                       sw.JointParams(dst[2], dst[3], dst[4]), sw.OutputParams(dst[5], dst[6]))
    e.close()
    g = grads(r)
    for k in O.GRAD_KEYS:
        assert np.array_equal(g[k], ref[k]), k
