"""GPU: the engine's scheduling knobs change only the order of work, never the
result. Each knob is read once per process, so each configuration runs in a
subprocess (tests/_knob_run.py) on the same inputs and is compared with the
float64 oracle and with the default schedule.

  SWTB_PARTS        parts a launch group is cut into (wavefront overlap)
  SWTB_LEAD         tile fraction of the lead part
  SWTB_JOINT_BATCH  launch groups per joint-network GEMM batch
  SWTB_CTA_GROUP    1-SM vs 2-SM (CTA pair) output-layer GEMMs (the dz GEMM
                    always runs as pairs)
  SWTB_LAT_W        multi-warp vs single-warp wavefront
  SWTB_LAT_PAIR     both wavefront directions of a sample in one CTA or two
  SWTB_DETERMINISTIC ordered split-K reductions vs fp32 atomics
  SWTB_BWD_SLAB_MB  backward sub-slab bound (1 MB: one 64-tile sub-slab each)
  SWTB_STORE_X      16-bit modes: dh from the forward's stored fp16 logits (x
                    slab) vs the logit-recompute GEMM

Also runs the C++ drop-in parity driver (oracle/_ref/ref_parity: the
unmodified reference engine and libswt_b200 through include/swt_b200.hpp in
one binary) when it was built."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RUNNER = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_knob_run.py")

sys.path.insert(0, ROOT)
from oracle import swt_oracle as O  # noqa: E402

KNOBS = [
    {},
    {"SWTB_PARTS": "1"},
    {"SWTB_PARTS": "3"},
    {"SWTB_LEAD": "0.5"},
    {"SWTB_JOINT_BATCH": "1"},
    {"SWTB_CTA_GROUP": "1"},
    {"SWTB_LAT_W": "1"},
    {"SWTB_LAT_PAIR": "1"},
    {"SWTB_DETERMINISTIC": "0"},
    {"SWTB_BWD_SLAB_MB": "1"},
]


def run(env_extra, tmp_path, tag, prec="tf32"):
    out = os.path.join(tmp_path, f"{tag}.npz")
    env = dict(os.environ)
    env.update(env_extra)
    subprocess.run([sys.executable, RUNNER, out, prec], check=True, env=env, cwd=ROOT,
                   timeout=600)
    return dict(np.load(out))


@pytest.fixture(scope="module")
def reference(tmp_path_factory):
    tmp = str(tmp_path_factory.mktemp("knobs"))
    base = run({}, tmp, "base")
    inp = dict(np.load(os.path.join(tmp, "base.npz.inputs.npz")))
    return tmp, base, O.run_step(inp)


@pytest.mark.parametrize("knob", KNOBS[1:], ids=lambda k: ",".join(f"{a}={b}" for a, b in k.items()))
def test_schedule_knob_invariance(reference, knob):
    tmp, base, ref = reference
    r = run(knob, tmp, "_".join(f"{a}{b}" for a, b in knob.items()))
    # same arithmetic, different order of fp32 accumulation only
    assert abs(float(r["loss"]) - float(base["loss"])) <= 1e-6 * abs(float(base["loss"]))
    for k in O.GRAD_KEYS:
        assert O.rel_err(r[k], base[k]) < 2e-4, (knob, k)
        assert O.rel_err(r[k], ref[k]) < 1e-3, (knob, k)  # tf32 bound vs f64 oracle


def test_zero_tile_skip_over_many_compacted_chunks(reference):
    """fp16 zero-tile skip with 1 MB backward sub-slabs: each part's active
    list is walked in many compacted chunks of 64 tiles (list offsets, the
    chunks past the device-side count launch empty) — same result as one
    chunk, and as the dense backward, within fp32 summation order."""
    tmp, _, ref = reference
    a = run({}, tmp, "skip_one", "fp16")
    b = run({"SWTB_BWD_SLAB_MB": "1"}, tmp, "skip_many", "fp16")
    c = run({"SWTB_SKIP_ZERO_TILES": "0"}, tmp, "skip_dense", "fp16")
    for r in (b, c):
        assert abs(float(r["loss"]) - float(a["loss"])) <= 1e-6 * abs(float(a["loss"]))
        for k in O.GRAD_KEYS:
            assert O.rel_err(r[k], a[k]) < 1e-4, k
    for k in O.GRAD_KEYS:
        assert O.rel_err(a[k], ref[k]) < 1e-3, k


@pytest.mark.parametrize("prec", ["fp16", "bf16x", "bf16"])
def test_store_x_matches_recompute(reference, prec):
    """dh formed from the forward's stored fp16 logits (SWTB_STORE_X=1, the
    alternative pipeline) against the logit-recompute GEMM (the default):
    both inside the mode's bound against the f64 oracle, and close to each
    other."""
    tmp, _, ref = reference
    a = run({"SWTB_STORE_X": "1"}, tmp, f"x_{prec}", prec)
    b = run({"SWTB_STORE_X": "0"}, tmp, f"rc_{prec}", prec)
    bound = {"fp16": 1e-3, "bf16x": 5e-3, "bf16": 3e-2}[prec]
    for r in (a, b):
        assert abs(float(r["loss"]) - float(ref["loss"])) <= 5e-4 * abs(float(ref["loss"]))
        for k in O.GRAD_KEYS:
            assert O.rel_err(r[k], ref[k]) < bound, (prec, k, O.rel_err(r[k], ref[k]))
    # the same forward GEMM; the stored-logits epilogue keeps the running
    # maximum (the recompute pipeline's may drop it), so the fp32 log-sum-exp
    # rounds differently in the last bits
    assert abs(float(a["loss"]) - float(b["loss"])) <= 1e-6 * abs(float(b["loss"]))
    for k in O.GRAD_KEYS:
        assert O.rel_err(a[k], b[k]) < bound, (prec, k)


def test_cpp_dropin_parity_driver():
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_parity")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/ref_parity not built (needs /root/reference at build time)")
    p = subprocess.run([exe, "--quick"], capture_output=True, text=True, timeout=600)
    lines = [json.loads(l) for l in p.stdout.splitlines() if l.startswith("{")]
    assert p.returncode == 0, p.stdout[-2000:]
    assert lines[-1] == {"failures": 0}
    assert all(l.get("pass", True) for l in lines)
