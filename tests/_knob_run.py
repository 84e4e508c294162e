"""Helper for tests/test_gpu_schedule.py (not a test module): one step of a
ragged synthetic batch through libswt_b200 under the caller's environment
(scheduling knobs), results saved to argv[1] (+ the inputs beside it);
argv[2] optionally names the precision mode (default tf32)."""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2211_16270_b200 as sw  # noqa: E402

out = sys.argv[1]
# 12 samples, ramped lengths (U1 up to 81: the multi-warp wavefront); small
# groups so several launch groups, parts and joint batches are exercised
batch, jp, op = sw.synth_inputs(12, 90, 80, 96, 160, H_A=72, H_L=40, seed=7)
prec = sys.argv[2] if len(sys.argv) > 2 else "tf32"
eng = sw.Engine(0, getattr(sw.Precision, prec), group_cells=12000)
r = eng.run_step(batch, jp, op, sw.EngineConfig(mode=sw.EngineMode.sample_wise_pr_dp))
g = r.grads
np.savez(out, loss=r.loss, sample_losses=np.asarray(r.sample_losses),
         dw_acoustic=g.dw_acoustic, dw_label=g.dw_label, dbias=g.dbias,
         dw_out=g.dw_out, dbias_out=g.dbias_out, dacoustic=g.dacoustic,
         dlabel=g.dlabel, groups=r.stats["groups"])
np.savez(out + ".inputs.npz", acoustic=batch.acoustic, label=batch.label,
         labels=batch.labels, t_len=batch.t_len, u_len=batch.u_len,
         w_acoustic=jp.w_acoustic, w_label=jp.w_label, bias=jp.bias,
         w_out=op.w_out, bias_out=op.bias_out)
eng.close()
