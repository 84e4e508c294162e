"""Small steps for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): config c1 shapes plus a ragged batch, every precision, the
sample-wise and batched modes, host and device buffers."""
import sys
import os

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2211_16270_b200 as sw  # noqa: E402

precs = [sw.Precision[p] for p in (sys.argv[1].split(",") if len(sys.argv) > 1 else
                                   ["fp16", "tf32", "bf16x", "bf16"])]
for prec in precs:
    e = sw.Engine(0, prec)
    # the third case has lattices long enough for the fp16 zero-tile skip to
    # leave tiles out of the backward (active-tile lists, row-mapped GEMMs)
    for B, T, U, H, V, ha, hl in ((2, 50, 10, 64, 32, 64, 64), (3, 37, 7, 96, 130, 40, 24),
                                  (2, 300, 60, 64, 96, 64, 64)):
        batch, jp, op = sw.synth_inputs(B, T, U, H, V, H_A=ha, H_L=hl)
        for mode in (sw.EngineMode.sample_wise_pr_dp, sw.EngineMode.batched):
            if T > 100 and mode == sw.EngineMode.batched:
                continue
            r = e.run_step(batch, jp, op, sw.EngineConfig(mode=mode))
            assert np.isfinite(r.loss)
            print(prec.name, B, T, U, mode.name, r.loss, "active tiles",
                  r.stats.get("active_tiles"), "of", r.stats.get("tiles"), flush=True)
    e.close()
print("sanitize case done")
