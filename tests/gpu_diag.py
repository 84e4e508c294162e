"""GPU bring-up diagnostics (prints, never asserts): each tcgen05 GEMM
majorness/precision combo vs torch fp32, the lattice op vs the CPU oracle,
and one small engine step vs the oracle."""
import sys, os, time, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2211_16270_b200 as sw
from oracle import swt_oracle as O

eng = sw.Engine(0, sw.Precision.bf16)
print("ctx ok; sms", torch.cuda.get_device_properties(0).multi_processor_count, flush=True)

def gemm_case(prec, a_mn, b_mn, M, N, K, acc=False):
    g = torch.Generator(device="cuda").manual_seed(0)
    dt = torch.bfloat16 if prec == sw.Precision.bf16 else torch.float32
    def mk(r, c):
        cp = (c + 31) // 32 * 32
        return torch.randn((r, cp), device="cuda", generator=g).to(dt)[:, :c]
    A = mk(K, M) if a_mn else mk(M, K)
    Bm = mk(K, N) if b_mn else mk(N, K)
    out = torch.zeros(M, N, device="cuda")
    if acc:
        out += 1.0
    eng.debug_gemm(A, Bm, out, a_mn=a_mn, b_mn=b_mn, precision=prec, accumulate=acc)
    Af = (A.float().t() if a_mn else A.float())
    Bf = (Bm.float() if b_mn else Bm.float().t())
    if prec == sw.Precision.tf32:
        Af = Af.view(torch.int32).bitwise_and(-8192).view(torch.float32)
        Bf = Bf.view(torch.int32).bitwise_and(-8192).view(torch.float32)
    ref = Af.double() @ Bf.double()
    if acc:
        ref += 1.0
    err = ((out.double() - ref).abs().max() / ref.abs().max()).item()
    return err

for prec in (sw.Precision.bf16, sw.Precision.tf32):
    for a_mn in (False, True):
        for b_mn in (False, True):
            for (M, N, K) in ((128, 256, 64), (300, 520, 200), (1000, 33, 515)):
                try:
                    e = gemm_case(prec, a_mn, b_mn, M, N, K)
                    e2 = gemm_case(prec, a_mn, b_mn, M, N, K, acc=True)
                    print(f"gemm {prec.name} a_mn={int(a_mn)} b_mn={int(b_mn)} {M}x{N}x{K}: store {e:.2e} atomic {e2:.2e}", flush=True)
                except Exception as ex:
                    print("gemm FAIL", prec.name, a_mn, b_mn, M, N, K, ex, flush=True)

# raw GEMM throughput (CUDA events on the engine's stream)
def timed(fn, iters=20):
    st = torch.cuda.ExternalStream(eng.stream)
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(iters):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters
for prec in (sw.Precision.bf16, sw.Precision.tf32):
    dt = torch.bfloat16 if prec == sw.Precision.bf16 else torch.float32
    for (M, N, K, a_mn, b_mn, acc) in ((65536, 1024, 512, 0, 0, 0), (65536, 512, 1024, 0, 1, 0), (1024, 512, 65536, 1, 1, 1)):
        A = torch.randn((K, M) if a_mn else (M, K), device="cuda").to(dt)
        Bm = torch.randn((K, N) if b_mn else (N, K), device="cuda").to(dt)
        out = torch.zeros(M, N, device="cuda")
        try:
            ms = timed(lambda: eng.debug_gemm(A, Bm, out, a_mn=bool(a_mn), b_mn=bool(b_mn), precision=prec, accumulate=bool(acc)), 10)
            print(f"perf {prec.name} {M}x{N}x{K} a_mn={a_mn} b_mn={b_mn} acc={acc}: {ms:.3f} ms (incl. sync) {2*M*N*K/ms/1e9:.1f} TFLOP/s", flush=True)
        except Exception as ex:
            print("perf FAIL", ex, flush=True)

# lattice op (f^W on explicit scores)
try:
    rng = np.random.default_rng(0)
    for (T, U, V) in ((1, 0, 2), (4, 2, 5), (50, 10, 32), (300, 80, 16)):
        s = rng.uniform(-2, 2, size=(T, U + 1, V))
        y = rng.integers(1, V, size=U)
        l_ref, d_ref = O.transducer_loss_sample(s, y)
        l, d = eng.transducer_loss_sample(s, y)
        print(f"fW T={T} U={U} V={V}: loss {l:.9f} ref {l_ref:.9f} rel {abs(l-l_ref)/abs(l_ref):.2e} dscores {O.rel_err(d, d_ref):.2e}", flush=True)
except Exception:
    traceback.print_exc()

# engine step
for prec in (sw.Precision.tf32, sw.Precision.bf16):
    for cfg in ((1, 50, 10, 64, 32), (4, 37, 9, 40, 50), (8, 64, 20, 128, 256)):
        try:
            e = sw.Engine(0, prec)
            B, T, U, H, V = cfg
            batch, jp, op = sw.synth_inputs(B, T, U, H, V)
            inp = dict(acoustic=batch.acoustic, label=batch.label, labels=batch.labels,
                       t_len=batch.t_len, u_len=batch.u_len, w_acoustic=jp.w_acoustic,
                       w_label=jp.w_label, bias=jp.bias, w_out=op.w_out, bias_out=op.bias_out)
            ref = O.run_step(inp)
            t0 = time.time()
            r = e.run_step(batch, jp, op)
            dt = time.time() - t0
            msg = " ".join(f"{k}={O.rel_err(getattr(r.grads, k), ref[k]):.1e}" for k in O.GRAD_KEYS)
            print(f"step {prec.name} {cfg}: loss {r.loss:.6f} ref {ref['loss']:.6f} rel {abs(r.loss-ref['loss'])/ref['loss']:.1e} | {msg} | {dt*1e3:.1f} ms {r.stats}", flush=True)
        except Exception:
            traceback.print_exc()
print("diag done", flush=True)
