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
