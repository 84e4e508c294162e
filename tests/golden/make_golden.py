"""Regenerates the committed golden fixtures in tests/golden/ by running the
UNMODIFIED reference engine (oracle/_ref/libswt_ref.so, compiled from
/root/reference by oracle/Makefile). Run in the dev container:

    make -C oracle ref && python tests/golden/make_golden.py

Fixtures (all outputs from the reference itself):
  fw.npz       f^W instances: scores, labels -> loss, dscores (f64)
               (transducer_loss_sample, loss.cpp:176-185) + path-enumeration
               losses (oracle.cpp:65-85)
  c1.npz       config c1 (B=1 T=50 U=10 V=32 H=64, seed 1): run_step<double>
               on the f32 inputs widened, and run_step<float>
  ragged.npz   a ragged batch with t_len=1 / u_len=0 / full-length samples and
               H_A != H_L != H: inputs + run_step<double> outputs
  meta.json    sha256 of synth_inputs arrays for c2/c3, padded_lengths and
               Eq. 9 tables, count_paths values
"""

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import ref as R  # noqa: E402

KEYS = ("loss", "sample_losses", "dw_acoustic", "dw_label", "dbias", "dw_out",
        "dbias_out", "dacoustic", "dlabel")


def fw():
    rng = np.random.default_rng(2211)
    out = {}
    cases = [(1, 0, 2), (2, 1, 2), (3, 2, 4), (4, 2, 5), (5, 3, 4), (2, 5, 7),
             (1, 4, 3), (6, 0, 3), (7, 3, 6), (5, 2, 9)]
    for i, (T, U, V) in enumerate(cases):
        s = rng.uniform(-2, 2, size=(T, U + 1, V))
        y = rng.integers(1, V, size=U).astype(np.int32)
        loss, ds = R.transducer_loss_sample(s, y)
        out[f"s{i}"] = s
        out[f"y{i}"] = y
        out[f"loss{i}"] = np.array(loss)
        out[f"ds{i}"] = ds
        out[f"enum{i}"] = np.array(R.enumerate_paths_loss(s, y))
    out["n"] = np.array(len(cases))
    np.savez_compressed(os.path.join(HERE, "fw.npz"), **out)


def c1():
    inp = R.synth_inputs(1, 50, 10, 64, 32)
    r64 = R.run_step(inp, dtype=np.float64)
    r32 = R.run_step(inp, dtype=np.float32)
    d = {f"f64_{k}": np.asarray(r64[k]) for k in KEYS}
    d.update({f"f32_{k}": np.asarray(r32[k]) for k in KEYS})
    np.savez_compressed(os.path.join(HERE, "c1.npz"), **d)


def ragged():
    inp = R.synth_inputs(6, 13, 5, 12, 9, H_A=7, H_L=5, seed=31)
    inp["t_len"] = np.array([13, 1, 7, 13, 2, 9], dtype=np.int64)
    inp["u_len"] = np.array([5, 0, 3, 0, 5, 1], dtype=np.int64)
    rng = np.random.default_rng(5)
    for b in range(6):
        inp["acoustic"][b, inp["t_len"][b]:] = 0
        inp["label"][b, inp["u_len"][b] + 1:] = 0
        inp["labels"][b, :] = 0
        inp["labels"][b, :inp["u_len"][b]] = rng.integers(1, 9, inp["u_len"][b])
    r = R.run_step(inp, dtype=np.float64, mode="sample_wise_pr_dp", workers=3)
    d = {f"in_{k}": v for k, v in inp.items()}
    d.update({f"f64_{k}": np.asarray(r[k]) for k in KEYS})
    np.savez_compressed(os.path.join(HERE, "ragged.npz"), **d)


def meta():
    m = {"synth_sha256": {}}
    for name, cfg in {"c2": (32, 200, 50, 256, 512),
                      "c3_B16": (16, 500, 100, 512, 1024)}.items():
        d = R.synth_inputs(*cfg)
        m["synth_sha256"][name] = {
            "cfg": cfg,
            **{k: hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest()
               for k, v in d.items()}}
    m["pi_table"] = [[f, l, v, b, R.parallel_iterations(f, l, v, b)] for
                     (f, l, v, b) in [(500, 100, 4096, 10**9),
                                      (232, 46, 4096, 10**9),
                                      (50, 10, 4096, 10**9),
                                      (500, 100, 4096, 1000),
                                      (2, 2, 2, 10**9), (10, 10, 10, 8000),
                                      (1000, 201, 1024, 10**9),
                                      (200, 51, 512, 10**9),
                                      (500, 101, 1024, 10**9),
                                      (750, 151, 4096, 10**9)]]
    m["count_paths"] = [[f, l, int(R.lib().ref_count_paths(f, l))]
                        for f, l in [(1, 0), (2, 1), (5, 3), (4, 2), (10, 4)]]
    with open(os.path.join(HERE, "meta.json"), "w") as f:
        json.dump(m, f, indent=1)


if __name__ == "__main__":
    fw()
    c1()
    ragged()
    meta()
    print("golden fixtures written to", HERE)
