"""The 1D walker's short zero-code predicate (lorenzo.cu zero_code) against
the full quantizer (common.cuh quantize, predict.py:93-115 semantics) on 40M
randomised (value, prediction, bound) cases incl. ties and extreme bounds.
Both are restated in plain C with the device's rounding (no FMA contraction)."""
import os
import shutil
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(os.path.dirname(HERE), "scripts", "micro", "zero_code_check.c")


@pytest.mark.skipif(shutil.which("gcc") is None, reason="needs gcc")
def test_short_zero_code_matches_quantizer(tmp_path):
    exe = str(tmp_path / "zq")
    subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-o", exe, SRC, "-lm"])
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout
    assert "bad=0" in out.stdout
