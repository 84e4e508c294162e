"""CPU: pin the oracle (oracle/swt_oracle.*) against the reference's own
known-answer tests and against the committed golden fixtures produced by the
unmodified reference (tests/golden/make_golden.py), and — when the reference
was compiled here (oracle/_ref) — against the reference directly.

Mirrors proj/tests/test_loss.cpp, test_oracle.cpp, test_bench.cpp and
acceptance.cpp criteria 1, 4, 7."""

import hashlib
import json
import math
import os
import subprocess

import numpy as np
import pytest

from oracle import ref as R
from oracle import swt_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")
KEYS = ("loss", "sample_losses") + O.GRAD_KEYS


def closed_form(T, U, V):
    return (T + U) * math.log(V) - math.log(O.count_paths(T, U))


# --- test_loss.cpp ----------------------------------------------------------

@pytest.mark.parametrize("T,U,V", [(1, 0, 2), (2, 1, 2), (5, 3, 4), (10, 4, 8)])
def test_uniform_logits_closed_form(T, U, V):
    # test_loss.cpp:102-115, acceptance.cpp:313-334
    loss, _ = O.transducer_loss_sample(np.zeros((T, U + 1, V)), [1] * U)
    assert abs(loss - closed_form(T, U, V)) < 1e-12 * max(1, loss)


def test_single_forced_blank():
    # test_loss.cpp:69-76, 144-149
    s = np.zeros((1, 1, 2))
    den = O.log_denominator(s)
    a, b = O.forward_backward(s, den, [])
    assert a[0, 0] == 0.0
    assert abs(b[0, 0] - math.log(0.5)) < 1e-15
    loss, ds = O.transducer_loss_sample(s, [])
    assert abs(loss - math.log(2)) < 1e-15
    assert np.allclose(ds[0, 0], [-0.5, 0.5], atol=1e-15)


def test_two_paths_uniform():
    # test_loss.cpp:78-85
    s = np.zeros((2, 2, 2))
    _, b = O.forward_backward(s, O.log_denominator(s), [1])
    assert abs(b[0, 0] + math.log(4)) < 1e-12


def test_log_denominator_extremes():
    # test_loss.cpp:42-53
    assert np.allclose(O.log_denominator(np.zeros((2, 3, 4))), math.log(4))
    s = np.full((1, 1, 2), 1000.0)
    assert abs(O.log_denominator(s)[0, 0] - (1000 + math.log(2))) < 1e-9


def test_enumeration_matches_forward_backward():
    # acceptance.cpp:72-98 (criterion 1)
    rng = np.random.default_rng(50_000)
    for _ in range(200):
        T, U, V = rng.integers(1, 6), rng.integers(0, 4), rng.integers(2, 5)
        s = rng.uniform(-2, 2, (T, U + 1, V))
        y = rng.integers(1, V, U)
        loss, _ = O.transducer_loss_sample(s, y)
        assert abs(loss - O.enumerate_paths_loss(s, y)) <= 1e-9 * max(1, abs(loss))


def test_gradient_invariants():
    # columns sum to zero (test_loss.cpp:151-162); shift invariance (164-178)
    rng = np.random.default_rng(60)
    s = rng.uniform(-2, 2, (4, 4, 5))
    y = rng.integers(1, 5, 3)
    loss, ds = O.transducer_loss_sample(s, y)
    assert np.abs(ds.sum(-1)).max() < 1e-10
    shifted = s + rng.uniform(-5, 5, (4, 4, 1))
    assert abs(O.transducer_loss_sample(shifted, y)[0] - loss) < 1e-10


def test_gradient_matches_finite_differences():
    # test_loss.cpp:180-195, oracle.hpp:39-42 tolerance
    rng = np.random.default_rng(65)
    s = rng.uniform(-2, 2, (3, 3, 4))
    y = rng.integers(1, 4, 2)
    _, ds = O.transducer_loss_sample(s, y)
    eps = 1e-6
    for idx in np.ndindex(s.shape):
        p = s.copy(); p[idx] += eps
        m = s.copy(); m[idx] -= eps
        fd = (O.transducer_loss_sample(p, y)[0] - O.transducer_loss_sample(m, y)[0]) / (2 * eps)
        assert abs(ds[idx] - fd) < max(1e-6 * abs(ds[idx]), 1e-8) + 1e-9


def test_error_paths():
    # test_loss.cpp:250-287
    s = np.zeros((2, 2, 3))
    with pytest.raises(O.OracleInputError):
        O.transducer_loss_sample(s, [5])
    with pytest.raises(O.OracleInputError):
        O.transducer_loss_sample(s, [1, 2])
    with pytest.raises(O.OracleInputError):
        O.transducer_loss_sample(np.zeros((0, 2, 3)), [1])


# --- test_oracle.cpp / test_engine.cpp / test_bench.cpp ---------------------

def test_count_paths():
    assert [O.count_paths(*a) for a in [(1, 0), (2, 1), (5, 3), (4, 2)]] == [1, 2, 35, 10]
    assert O.count_paths(0, 2) == -1


def test_parallel_iterations_table():
    # acceptance.cpp:402-411, test_engine.cpp:48-58
    assert O.compute_parallel_iterations(500, 100, 4096, 10**9) == 1
    assert O.compute_parallel_iterations(232, 46, 4096, 10**9) == 4
    assert O.compute_parallel_iterations(50, 10, 4096, 10**9) == 16
    assert O.compute_parallel_iterations(500, 100, 4096, 1000) == 1
    assert O.compute_parallel_iterations(2, 2, 2, 10**9) == 16
    assert O.compute_parallel_iterations(10, 10, 10, 8000) == 2
    with pytest.raises(O.OracleInputError):
        O.compute_parallel_iterations(0, 1, 1, 100)


def test_padded_lengths():
    # test_bench.cpp:34-54
    t, u = O.padded_lengths(4, 500, 100)
    assert list(t) == [500, 485, 469, 454] and list(u) == [100, 85, 69, 54]
    t, u = O.padded_lengths(1, 500, 100)
    assert list(t) == [500] and list(u) == [100]
    for B in (1, 2, 3, 7, 64):
        t, u = O.padded_lengths(B, 37, 11)
        assert t[0] == 37 and u[0] == 11 and t.min() >= 1 and u.min() >= 1


def test_mt19937_64_standard_value():
    # ISO C++ [rand.predef]: the 10000th output of default-seeded mt19937_64
    assert int(O.mt19937_64(5489, 10000)[-1]) == 9981545732273789042


def test_synth_inputs_properties():
    # test_bench.cpp:56-97
    d = O.synth_inputs(4, 8, 3, 6, 8, H_A=5, H_L=5, seed=3)
    for b in range(4):
        assert np.all(d["acoustic"][b, d["t_len"][b]:] == 0)
        assert np.all(d["label"][b, d["u_len"][b] + 1:] == 0)
        labs = d["labels"][b, :d["u_len"][b]]
        assert np.all((labs >= 1) & (labs < 8))
    assert np.abs(d["acoustic"]).max() <= 0.1
    e = O.synth_inputs(4, 8, 3, 6, 8, H_A=5, H_L=5, seed=4)
    assert not np.array_equal(d["acoustic"], e["acoustic"])


# --- golden fixtures from the reference --------------------------------------

def test_fw_golden():
    g = np.load(os.path.join(GOLD, "fw.npz"))
    for i in range(int(g["n"])):
        loss, ds = O.transducer_loss_sample(g[f"s{i}"], g[f"y{i}"])
        assert abs(loss - float(g[f"loss{i}"])) <= 1e-12 * max(1, abs(loss))
        assert np.abs(ds - g[f"ds{i}"]).max() <= 1e-12
        assert abs(O.enumerate_paths_loss(g[f"s{i}"], g[f"y{i}"]) - float(g[f"enum{i}"])) <= 1e-12 * max(1, abs(loss))


def test_c1_golden():
    g = np.load(os.path.join(GOLD, "c1.npz"))
    out = O.run_step(O.synth_inputs(1, 50, 10, 64, 32))
    assert abs(out["loss"] - float(g["f64_loss"])) <= 1e-12 * out["loss"]
    for k in O.GRAD_KEYS:
        assert O.rel_err(out[k], g[f"f64_{k}"]) < 1e-12, k
    # the reference's own f32 path vs its f64 path
    for k in O.GRAD_KEYS:
        assert O.rel_err(g[f"f32_{k}"], g[f"f64_{k}"]) < 1e-4, k


def test_ragged_golden():
    g = np.load(os.path.join(GOLD, "ragged.npz"))
    inp = {k[3:]: g[k] for k in g.files if k.startswith("in_")}
    out = O.run_step(inp)
    assert abs(out["loss"] - float(g["f64_loss"])) <= 1e-12 * out["loss"]
    for k in O.GRAD_KEYS + ("sample_losses",):
        assert O.rel_err(out[k], g[f"f64_{k}"]) < 1e-12, k
    # padding of the encoder-input gradients is exactly zero (test_engine.cpp:327-347)
    for b in range(6):
        assert np.all(out["dacoustic"][b, inp["t_len"][b]:] == 0)
        assert np.all(out["dlabel"][b, inp["u_len"][b] + 1:] == 0)


def test_synth_matches_reference_hashes():
    with open(os.path.join(GOLD, "meta.json")) as f:
        meta = json.load(f)
    for name, rec in meta["synth_sha256"].items():
        B, T, U, H, V = rec["cfg"]
        d = O.synth_inputs(B, T, U, H, V)
        for k, v in d.items():
            assert hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest() == rec[k], (name, k)
    for f, l, v, b, pi in meta["pi_table"]:
        assert O.compute_parallel_iterations(f, l, v, b) == pi
    for f, l, c in meta["count_paths"]:
        assert O.count_paths(f, l) == c


# --- the compiled reference itself (dev container) ----------------------------

needs_ref = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")


@needs_ref
def test_reference_acceptance_binary():
    out = subprocess.run([R.ACCEPTANCE], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout
    assert "10/10 criteria passed" in out.stdout


@needs_ref
def test_oracle_equals_reference_on_ragged_batches():
    rng = np.random.default_rng(70_000)
    for i in range(10):
        B, T, U = rng.integers(1, 6), rng.integers(1, 12), rng.integers(1, 6)
        H, HA, HL, V = rng.integers(1, 9), rng.integers(1, 7), rng.integers(1, 7), rng.integers(2, 7)
        inp = R.synth_inputs(B, T, U, H, V, H_A=HA, H_L=HL, seed=100 + i)
        inp["t_len"] = rng.integers(1, T + 1, B).astype(np.int64)
        inp["u_len"] = rng.integers(0, U + 1, B).astype(np.int64)
        for b in range(B):
            inp["acoustic"][b, inp["t_len"][b]:] = 0
            inp["label"][b, inp["u_len"][b] + 1:] = 0
            inp["labels"][b] = 0
            inp["labels"][b, :inp["u_len"][b]] = rng.integers(1, V, inp["u_len"][b])
        ref = R.run_step(inp, mode="sample_wise_pr_dp", workers=3)
        out = O.run_step(inp)
        assert abs(out["loss"] - ref["loss"]) <= 1e-12 * max(1, abs(ref["loss"]))
        for k in O.GRAD_KEYS:
            assert O.rel_err(out[k], ref[k]) < 1e-12, (i, k)


@needs_ref
def test_synth_bit_identical_to_reference():
    for cfg in [(1, 50, 10, 64, 32), (3, 20, 5, 8, 7), (32, 200, 50, 256, 512)]:
        a, b = R.synth_inputs(*cfg), O.synth_inputs(*cfg)
        for k in a:
            assert np.array_equal(a[k], b[k]), (cfg, k)
