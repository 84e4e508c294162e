"""GPU: the tcgen05 GEMM core and the f^W lattice kernels of libswt_b200,
called through the C ABI.

* GEMM: every operand majorness x precision combination, store and split-K
  atomic epilogues, ragged (non-tile-multiple) shapes, against a float64
  torch reference of the same rounded operands (tolerance 1e-5 normalized).
* f^W (swtb_transducer_loss, reference loss.cpp:176-185): the reference's
  own known-answer tests (test_loss.cpp, acceptance.cpp criteria 1 and 4) and
  the committed golden vectors produced by the reference (tests/golden/fw.npz).
  The GPU lattice accumulates in f64 with f32 transcendentals and f32
  log-softmax: tolerance 1e-6 relative on the loss, 1e-5 normalized on the
  score gradients (the reference's own f32 path is at ~1e-7 / 1e-6)."""

import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_2211_16270_b200 as sw  # noqa: E402
from oracle import swt_oracle as O  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def eng():
    e = sw.Engine(0, sw.Precision.bf16)
    yield e
    e.close()


def _operand(rows, cols, dt, g):
    cp = (cols + 31) // 32 * 32  # TMA needs 16-byte row pitch
    return torch.randn((rows, cp), device="cuda", generator=g).to(dt)[:, :cols]


@pytest.mark.parametrize("prec", [sw.Precision.bf16, sw.Precision.tf32])
@pytest.mark.parametrize("a_mn", [False, True])
@pytest.mark.parametrize("b_mn", [False, True])
@pytest.mark.parametrize("shape", [(128, 256, 64), (300, 520, 200),
                                   (1000, 33, 515), (7, 5, 3), (4096, 1024, 512)])
@pytest.mark.parametrize("acc", [False, True])
def test_gemm(eng, prec, a_mn, b_mn, shape, acc):
    M, N, K = shape
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N * 3 + K)
    dt = torch.bfloat16 if prec == sw.Precision.bf16 else torch.float32
    A = _operand(K, M, dt, g) if a_mn else _operand(M, K, dt, g)
    B = _operand(K, N, dt, g) if b_mn else _operand(N, K, dt, g)
    out = torch.full((M, N), 0.5 if acc else 0.0, device="cuda")
    eng.debug_gemm(A, B, out, a_mn=a_mn, b_mn=b_mn, precision=prec, accumulate=acc)
    Af = A.float().t() if a_mn else A.float()
    Bf = B.float() if b_mn else B.float().t()
    if prec == sw.Precision.tf32:  # the tensor core reads the tf32 subset
        Af = Af.view(torch.int32).bitwise_and(-8192).view(torch.float32)
        Bf = Bf.view(torch.int32).bitwise_and(-8192).view(torch.float32)
    ref = Af.double() @ Bf.double() + (0.5 if acc else 0.0)
    err = ((out.double() - ref).abs().max() / ref.abs().max()).item()
    assert err < 1e-5, err


# --- f^W ----------------------------------------------------------------------

@pytest.mark.parametrize("T,U,V", [(1, 0, 2), (2, 1, 2), (5, 3, 4), (10, 4, 8),
                                   (300, 60, 16)])
def test_uniform_logits_closed_form(eng, T, U, V):
    loss, _ = eng.transducer_loss_sample(np.zeros((T, U + 1, V)), [1] * U)
    cf = (T + U) * math.log(V) - math.log(math.comb(T + U - 1, U))
    assert abs(loss - cf) <= 1e-6 * max(1.0, cf)


def test_forced_blank_cell_gradient(eng):
    loss, ds = eng.transducer_loss_sample(np.zeros((1, 1, 2)), [])
    assert abs(loss - math.log(2)) < 1e-7
    assert np.allclose(ds[0, 0], [-0.5, 0.5], atol=1e-7)


def test_fw_golden(eng):
    g = np.load(os.path.join(GOLD, "fw.npz"))
    for i in range(int(g["n"])):
        loss, ds = eng.transducer_loss_sample(g[f"s{i}"], g[f"y{i}"])
        ref = float(g[f"loss{i}"])
        assert abs(loss - ref) <= 1e-6 * max(1.0, abs(ref)), i
        assert O.rel_err(ds, g[f"ds{i}"]) < 1e-5, i
        assert abs(loss - float(g[f"enum{i}"])) <= 1e-6 * max(1.0, abs(ref)), i


def test_path_enumeration_200_instances(eng):
    # acceptance.cpp criterion 1
    rng = np.random.default_rng(50_000)
    for _ in range(200):
        T, U, V = rng.integers(1, 6), rng.integers(0, 4), rng.integers(2, 5)
        s = rng.uniform(-2, 2, (T, U + 1, V))
        y = rng.integers(1, V, U)
        loss, _ = eng.transducer_loss_sample(s, y)
        ref = O.enumerate_paths_loss(s, y)
        assert abs(loss - ref) <= 1e-6 * max(1.0, abs(ref))


def test_finite_differences_50_instances(eng):
    # acceptance.cpp criterion 2 / test_loss.cpp FD checks, on the GPU f^W op.
    # The GPU lattice's loss is good to ~1e-6 relative (f32 transcendentals),
    # so the central difference uses eps = 1e-2: truncation + rounding stay
    # below 2e-3 absolute for these O(1) scores.
    rng = np.random.default_rng(20_000)
    eps = 1e-2
    for _ in range(50):
        T, U, V = rng.integers(1, 6), rng.integers(0, 4), rng.integers(2, 5)
        s = rng.uniform(-1, 1, (T, U + 1, V))
        y = rng.integers(1, V, U)
        _, ds = eng.transducer_loss_sample(s, y)
        for _ in range(4):
            idx = tuple(int(rng.integers(0, n)) for n in s.shape)
            sp, sm = s.copy(), s.copy()
            sp[idx] += eps
            sm[idx] -= eps
            fd = (eng.transducer_loss_sample(sp, y)[0] - eng.transducer_loss_sample(sm, y)[0]) / (2 * eps)
            assert abs(fd - ds[idx]) <= 2e-3 * max(1.0, abs(ds[idx])), (T, U, V, idx, fd, ds[idx])


def test_gradient_invariants(eng):
    rng = np.random.default_rng(60)
    s = rng.uniform(-2, 2, (40, 13, 9))
    y = rng.integers(1, 9, 12)
    loss, ds = eng.transducer_loss_sample(s, y)
    assert np.abs(ds.sum(-1)).max() < 1e-6           # test_loss.cpp:151-162
    shifted = s + rng.uniform(-5, 5, (40, 13, 1))     # test_loss.cpp:164-178
    assert abs(eng.transducer_loss_sample(shifted, y)[0] - loss) < 1e-5 * loss
    ref_loss, ref_ds = O.transducer_loss_sample(s, y)
    assert abs(loss - ref_loss) < 1e-6 * ref_loss
    assert O.rel_err(ds, ref_ds) < 1e-5


def test_many_labels_per_frame(eng):
    # U >> T is legal (test_loss.cpp:238-248); U+1 > 1024 takes the wide kernel
    rng = np.random.default_rng(71)
    for T, U in [(2, 5), (3, 40), (2, 1100)]:
        s = rng.uniform(-2, 2, (T, U + 1, 7))
        y = rng.integers(1, 7, U)
        loss, ds = eng.transducer_loss_sample(s, y)
        ref, rds = O.transducer_loss_sample(s, y)
        assert abs(loss - ref) <= 1e-6 * abs(ref)
        assert O.rel_err(ds, rds) < 1e-5


def test_long_lattice_matches_oracle(eng):
    rng = np.random.default_rng(3)
    s = rng.uniform(-1, 1, (1000, 201, 4))
    y = rng.integers(1, 4, 200)
    loss, ds = eng.transducer_loss_sample(s, y)
    ref, rds = O.transducer_loss_sample(s, y)
    assert abs(loss - ref) <= 1e-6 * abs(ref)
    assert O.rel_err(ds, rds) < 1e-5


def test_fw_error_paths(eng):
    with pytest.raises(sw.InvalidInputError):
        eng.transducer_loss_sample(np.zeros((2, 2, 3)), [5])       # label >= V
    with pytest.raises(sw.InvalidInputError):
        eng.transducer_loss_sample(np.zeros((2, 2, 3)), [0])       # blank label
    with pytest.raises(sw.InvalidInputError):
        eng.transducer_loss_sample(np.zeros((2, 2, 3)), [1, 2])    # count mismatch
    with pytest.raises(sw.InvalidInputError):
        eng.transducer_loss_sample(np.zeros((0, 2, 3)), [1])       # no frames
    with pytest.raises(sw.NumericalDegeneracyError):
        s = np.zeros((2, 2, 3))
        s[:, :, 0] = np.inf
        eng.transducer_loss_sample(s, [1])
