import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2211_16270_b200 as sw
from oracle import swt_oracle as O
batch, jp, op = sw.synth_inputs(8, 120, 30, 256, 512)
for prec in (sw.Precision.tf32, sw.Precision.bf16):
    eng = sw.Engine(0, prec)
    rs = [eng.run_step(batch, jp, op) for _ in range(4)]
    for k in O.GRAD_KEYS:
        e = max(O.rel_err(getattr(r.grads, k), getattr(rs[0].grads, k)) for r in rs[1:])
        if e > 1e-6: print(os.environ.get("SWTB_LIB"), prec.name, k, e)
    print(os.environ.get("SWTB_LIB"), prec.name, "losses", [r.loss for r in rs])
