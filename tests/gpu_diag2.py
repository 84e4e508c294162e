import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2211_16270_b200 as sw
from oracle import swt_oracle as O
def case(B,T,U,H,HA,HL,V,seed,t_len=None,u_len=None,labels=None):
    d = O.synth_inputs(B,T,U,H,V,H_A=HA,H_L=HL,seed=seed)
    if t_len is not None:
        d["t_len"]=np.array(t_len,np.int64); d["u_len"]=np.array(u_len,np.int64)
        for b in range(B):
            d["acoustic"][b,d["t_len"][b]:]=0; d["label"][b,d["u_len"][b]+1:]=0
            d["labels"][b]=0; d["labels"][b,:d["u_len"][b]]=labels[b][:d["u_len"][b]]
    return d
rng = np.random.default_rng(70_000)
for i in range(8):
    B, T, U = rng.integers(1, 9), rng.integers(1, 40), rng.integers(1, 12)
    H, HA, HL, V = rng.integers(1, 70), rng.integers(1, 40), rng.integers(1, 40), rng.integers(2, 90)
    tl = rng.integers(1, T + 1, B); ul = rng.integers(0, U + 1, B)
    labs = [rng.integers(1, V, ul[b]) for b in range(B)]
d = case(int(B),int(T),int(U),int(H),int(HA),int(HL),int(V),907,tl,ul,labs)
print("case", B,T,U,H,HA,HL,V, tl, ul)
ref = O.run_step(d)
print("oracle", ref["sample_losses"])
for prec in (sw.Precision.tf32, sw.Precision.bf16):
    for gc in (0, 1):
        e = sw.Engine(0, prec, group_cells=gc)
        b = sw.Batch(d["acoustic"], d["label"], d["labels"], d["t_len"], d["u_len"])
        r = e.run_step(b, sw.JointParams(d["w_acoustic"], d["w_label"], d["bias"]), sw.OutputParams(d["w_out"], d["bias_out"]))
        print(prec.name, "group_cells", gc, np.asarray(r.sample_losses) - ref["sample_losses"], r.stats["groups"])
# variants: V=3, and same with H=64
for (H2, V2) in ((40, 3), (64, 2), (40, 2)):
    d = case(3, 14, 3, H2, 26, 27, V2, 5)
    ref = O.run_step(d)
    for prec in (sw.Precision.tf32, sw.Precision.bf16):
        e = sw.Engine(0, prec)
        b = sw.Batch(d["acoustic"], d["label"], d["labels"], d["t_len"], d["u_len"])
        r = e.run_step(b, sw.JointParams(d["w_acoustic"], d["w_label"], d["bias"]), sw.OutputParams(d["w_out"], d["bias_out"]))
        print("H",H2,"V",V2, prec.name, np.asarray(r.sample_losses) - ref["sample_losses"])
