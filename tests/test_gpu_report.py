"""GPU: report.py sweeps through libswt_b200 in the reference's report schema
(bench.cpp:171-298): bare-T length sweep with U scaled, JSON read back."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_length_sweep_report():
    out = subprocess.run(
        [sys.executable, os.path.join(ROOT, "report.py"), "sweep", "--axis", "lengths",
         "--values", "20,40", "--batch", "2", "--frames", "40", "--labels", "8",
         "--joint", "64", "--vocab", "64", "--steps", "2", "--warmup", "1",
         "--format", "json"], check=True, capture_output=True, text=True, timeout=600).stdout
    rows = json.loads(out)
    assert [(r["T"], r["U"]) for r in rows] == [(20, 4), (40, 8)]
    for r in rows:
        assert r["status"] == "ok" and r["precision"] == "f32"
        assert r["operand_precision"] == "fp16"
        assert r["median_step_seconds"] > 0 and r["peak_bytes"] > 0
        assert r["loss_checksum"] > 0


def test_descending_sweep_exits_2():
    p = subprocess.run([sys.executable, os.path.join(ROOT, "report.py"), "sweep",
                        "--axis", "batch", "--values", "4,2"], capture_output=True, text=True)
    assert p.returncode == 2 and "ascend" in p.stderr
