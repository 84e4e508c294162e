"""CPU, world_size 2 over gloo: the multi-GPU contract of libswt_b200 —
sample b is processed by rank b % N, the theta-grads and the per-sample loss
vector are summed with ONE all-reduce, and each rank owns only its samples'
dh^A / dh^L slots — reproduces the single-process reference step exactly.
The oracle stands in for each rank's device work; the collective is real."""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import swt_oracle as O

THETA = ("dw_acoustic", "dw_label", "dbias", "dw_out", "dbias_out")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    inp = O.synth_inputs(5, 12, 4, 8, 9, H_A=6, H_L=7, seed=11)
    B = 5
    shard = list(range(rank, B, world))          # libswt_b200 make_plan
    part = O.run_step(inp, samples=shard)
    # one packed buffer, one all-reduce (swtb_engine.cpp "theta" layout)
    flat = np.concatenate([part[k].ravel() for k in THETA] + [part["sample_losses"]])
    t = torch.from_numpy(flat.copy())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    red = t.numpy()
    out, off = {}, 0
    for k in THETA:
        n = part[k].size
        out[k] = red[off:off + n].reshape(part[k].shape)
        off += n
    out["sample_losses"] = red[off:]
    out["loss"] = float(np.sum(out["sample_losses"]))  # ascending-b host sum
    owned_ok = all(np.all(part["dacoustic"][b] == 0) for b in range(B) if b not in shard)
    q.put((rank, out, part["dacoustic"], part["dlabel"], shard, owned_ok))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharded_step_equals_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = O.run_step(O.synth_inputs(5, 12, 4, 8, 9, H_A=6, H_L=7, seed=11))
    dac = np.zeros_like(full["dacoustic"])
    dlb = np.zeros_like(full["dlabel"])
    for rank, out, pa, pl, shard, owned_ok in res:
        assert owned_ok
        for k in THETA + ("sample_losses",):
            assert O.rel_err(out[k], full[k]) < 1e-12, (rank, k)
        assert abs(out["loss"] - full["loss"]) < 1e-9 * full["loss"]
        for b in shard:
            dac[b] = pa[b]
            dlb[b] = pl[b]
    assert O.rel_err(dac, full["dacoustic"]) < 1e-12
    assert O.rel_err(dlb, full["dlabel"]) < 1e-12
