"""CPU: report.py emits the reference's report schema
(proj/core/src/bench.cpp:249-298) — CSV columns in order, %.17g step
seconds, JSON with loss_checksum; empty reports are refused."""

import json

import pytest

import report


def _row(**kw):
    r = dict(mode="sample_wise_pr_dp", B=2, T=50, U=10, H=64, H_A=64, H_L=64, V=32,
             precision="bf16", median_step_seconds=0.1, peak_bytes=123, status="ok",
             seed=1, loss_checksum=178.5)
    r.update(kw)
    return r


def test_csv_schema_matches_reference():
    out = report.emit([_row(), _row(B=4, status="oom")], "csv").splitlines()
    assert out[0] == "mode,B,T,U,H,H_A,H_L,V,precision,median_step_seconds,peak_bytes,status,seed"
    assert out[1] == "sample_wise_pr_dp,2,50,10,64,64,64,32,bf16,0.10000000000000001,123,ok,1"
    assert out[2].split(",")[11] == "oom"


def test_json_schema_matches_reference():
    j = json.loads(report.emit([_row()], "json"))
    assert list(j[0]) == list(report.COLUMNS) + ["loss_checksum"]
    assert j[0]["loss_checksum"] == 178.5


def test_empty_report_refused():
    with pytest.raises(ValueError):
        report.emit([], "csv")


# --- sweep parsing (reference bench.cpp:171-221, test_bench.cpp cases) -------

def test_sweep_batch_axis():
    assert report.parse_sweep_values((8, 64, 16), "batch", "1,2,4") == [
        (1, 64, 16), (2, 64, 16), (4, 64, 16)]


def test_sweep_lengths_txu_and_bare_t_scaling():
    pts = report.parse_sweep_values((4, 1000, 200), "lengths", "50x10,250,500,1000")
    # bare T scales U by T / T_base, rounded half away from zero
    assert pts == [(4, 50, 10), (4, 250, 50), (4, 500, 100), (4, 1000, 200)]
    assert report.parse_sweep_values((4, 1000, 3), "lengths", "100")[0] == (4, 100, 1)


@pytest.mark.parametrize("axis,values,msg", [
    ("batch", "4,2", "ascend"), ("lengths", "50x10,50x20", "ascend"),
    ("batch", "0", "out of range"), ("lengths", "10x0", "out of range"),
    ("batch", "a", "cannot parse"), ("batch", ",,", "at least one"),
])
def test_sweep_rejections(axis, values, msg):
    with pytest.raises(report.InvalidInputError, match=msg):
        report.parse_sweep_values((8, 64, 16), axis, values)


def test_precision_field_reads_back_as_f32():
    # the reference's parse_report_json maps anything but "f32" to f64
    j = json.loads(report.emit([_row(precision="f32", operand_precision="fp16")], "json"))
    assert j[0]["precision"] == "f32" and j[0]["operand_precision"] == "fp16"
