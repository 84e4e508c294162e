import sys, time, json
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2211_16270_b200 as sw
B,T,U,H,V = 1024,1000,200,512,1024
batch, jp, op = sw.synth_inputs(B,T,U,H,V, seed=1)
eng = sw.Engine(0, sw.Precision.bf16)
cfg = sw.EngineConfig(mode=sw.EngineMode.sample_wise_pr_dp)
d = lambda x: torch.from_numpy(x).cuda()
db = sw.Batch(d(batch.acoustic), d(batch.label), d(batch.labels), batch.t_len, batch.u_len)
djp = sw.JointParams(d(jp.w_acoustic), d(jp.w_label), d(jp.bias)); dop = sw.OutputParams(d(op.w_out), d(op.bias_out))
z = lambda *s: torch.empty(*s, dtype=torch.float32, device='cuda')
dout = sw.GradientSet(z(H,H), z(H,H), z(H), z(V,H), z(V), z(B,T,H), z(B,U+1,H)); dsl = z(B)
pin = lambda x: torch.from_numpy(x).pin_memory().numpy()
hb = sw.Batch(pin(batch.acoustic), pin(batch.label), pin(batch.labels), batch.t_len, batch.u_len)
hjp = sw.JointParams(pin(jp.w_acoustic), pin(jp.w_label), pin(jp.bias)); hop = sw.OutputParams(pin(op.w_out), pin(op.bias_out))
hz = lambda *s: torch.empty(*s, dtype=torch.float32).pin_memory().numpy()
hout = sw.GradientSet(hz(H,H), hz(H,H), hz(H), hz(V,H), hz(V), hz(B,T,H), hz(B,U+1,H)); hsl = np.empty(B, np.float32)
def run(tag, f, n=3):
    f(); torch.cuda.synchronize()
    eng.set_profiling(True); eng.profile(reset=True)
    t0=time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize(); dt=(time.perf_counter()-t0)/n
    p=eng.profile(reset=True); eng.set_profiling(False)
    print(tag, round(dt*1e3,1), {k: round(v[0]/n,1) for k,v in p.items() if v[0]>0})
for _ in range(2):
    run('device', lambda: eng.run_step(db, djp, dop, cfg, out=dout, sample_losses=dsl))
    run('host  ', lambda: eng.run_step(hb, hjp, hop, cfg, out=hout, sample_losses=hsl))
    run('hin   ', lambda: eng.run_step(hb, hjp, hop, cfg, out=dout, sample_losses=dsl))
