"""The short zero-code predicate (a zero code needs floor(|q|) == 0, so only
|q| near 0.5 needs the tie re-division) against the full quantizer
(common.cuh quantize, predict.py:93-115 semantics) on 40M randomised (value,
prediction, bound) cases incl. ties and extreme bounds -- the condition the
1D walker's inner zero-code interval (lorenzo.cu zinner) is a subset of.
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
