"""CPU: the drop-in boundary. libswt_b200.so loads, exports every entry point
include/swt_b200.h declares, its host-only helpers agree with the oracle /
reference, errors map onto the reference exception types, and without a GPU
there is no silent CPU path (context creation fails loudly)."""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2211_16270_b200 as sw
from oracle import swt_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "swt_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(swtb_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_abi():
    fns = declared_functions()
    assert "swtb_step" in fns and "swtb_ctx_create" in fns
    assert set(fns) == set(sw.ABI_SYMBOLS), set(fns) ^ set(sw.ABI_SYMBOLS)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(sw.LIB_PATH)
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", sw.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\b(swtb_[a-z0-9_]+)\b", out))
    assert set(declared_functions()) <= exported


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", sw.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", sw.LIB_PATH],
                          capture_output=True, text=True).stdout
    # tcgen05 MMAs, TMEM loads and TMA loads are in the binary
    assert "UTCHMMA" in sass and "LDTM" in sass and "UTMALDG" in sass


def test_abi_version():
    assert sw.abi_version() == 3


def test_parallel_iterations_matches_reference_table():
    for f, l, v, b in [(500, 100, 4096, 10**9), (232, 46, 4096, 10**9),
                       (50, 10, 4096, 10**9), (500, 100, 4096, 1000),
                       (2, 2, 2, 10**9), (10, 10, 10, 8000),
                       (1000, 201, 1024, 10**9), (10**6, 10**6, 10**6, 10**9)]:
        assert sw.compute_parallel_iterations(f, l, v, b) == \
            O.compute_parallel_iterations(f, l, v, b)
    with pytest.raises(sw.InvalidInputError):
        sw.compute_parallel_iterations(0, 1, 1, 100)


def test_padded_lengths_match():
    for B, T, U in [(4, 500, 100), (1, 500, 100), (1024, 1000, 200), (7, 37, 11)]:
        a = sw.padded_lengths(B, T, U)
        b = O.padded_lengths(B, T, U)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    with pytest.raises(sw.InvalidInputError):
        sw.padded_lengths(0, 5, 5)


@pytest.mark.parametrize("cfg", [(1, 50, 10, 64, 32), (3, 20, 5, 8, 7),
                                 (32, 200, 50, 256, 512)])
def test_synth_inputs_bit_identical(cfg):
    B, T, U, H, V = cfg
    batch, jp, op = sw.synth_inputs(B, T, U, H, V)
    o = O.synth_inputs(B, T, U, H, V)
    got = dict(acoustic=batch.acoustic, label=batch.label, labels=batch.labels,
               t_len=batch.t_len, u_len=batch.u_len, w_acoustic=jp.w_acoustic,
               w_label=jp.w_label, bias=jp.bias, w_out=op.w_out,
               bias_out=op.bias_out)
    for k, v in o.items():
        assert np.array_equal(v, got[k]), k


def test_synth_rejects_bad_config():
    with pytest.raises(sw.InvalidInputError):
        sw.synth_inputs(1, 5, 2, 4, 1)


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback_without_gpu():
    with pytest.raises(sw.CudaError):
        sw.Engine(0)
