"""The drop-in proof: the UNMODIFIED reference package (fzpipe, installed in
baseline/_ref by scripts/install_reference.sh) runs its own pipeline with
this package's GPU modules plugged in (paper_2509_20563_b200.plugin), and
  * its archives at full-size C1/C3 equal fzpipe's own bytes (the SHA-256
    goldens made without the plugin), with the plugin's call counters
    proving the kernels ran;
  * its own test suite (test_pipeline.py, test_predict.py, test_encode.py,
    test_acceptance.py) passes with the plugin installed.
Skipped when baseline/_ref is absent (it is git-ignored; gpurun ships it).
"""

import hashlib
import json
import os
import subprocess
import sys

import pytest

from conftest import GOLDEN, ROOT

REF = os.path.join(ROOT, "baseline", "_ref")
pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)
if not os.path.isdir(os.path.join(REF, "fzpipe")):
    pytest.skip("reference not installed in baseline/_ref (scripts/install_reference.sh)", allow_module_level=True)

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/fzpipe_numba_cache")
if REF not in sys.path:
    sys.path.insert(0, REF)

G = json.load(open(os.path.join(GOLDEN, "fullsize.json")))


@pytest.fixture
def plugged():
    import fzpipe  # noqa: F401
    from paper_2509_20563_b200 import plugin
    plugin.install()
    plugin.calls.clear()
    yield plugin
    plugin.uninstall()


@pytest.mark.parametrize("case,preset", [("c1", "default"), ("c1", "speed"), ("c1", "quality"), ("c3", "quality")])
def test_fzpipe_pipeline_with_plugin_is_byte_identical(plugged, case, preset):
    import fzpipe
    from fzpipe.data import SyntheticSpec, generate
    e = G[case]
    f = generate(SyntheticSpec(e["kind"], tuple(e["dims"]), e["seed"]))
    eb = fzpipe.ErrorBoundSpec(fzpipe.ErrorMode.VALUE_RANGE_RELATIVE, e["rel_eb"])
    a = fzpipe.compress(f, eb, preset)            # fzpipe's own executor, GPU modules underneath
    blob = fzpipe.serialize_archive(a)
    want = e["archives"][preset]
    assert hashlib.sha256(blob).hexdigest() == want["archive_sha256"]
    r = fzpipe.decompress(fzpipe.parse_archive(blob))
    assert hashlib.sha256(r.data.tobytes()).hexdigest() == want["recon_sha256"]
    pred = "interp_quantize" if preset == "quality" else "lorenzo_quantize"
    codec = "bitshuffle_encode" if preset == "speed" else "huffman_encode"
    assert plugged.calls[pred] == 1 and plugged.calls[codec] == 1, dict(plugged.calls)


def test_reference_test_suite_passes_with_plugin():
    tests = os.path.join(REF, "fzpipe_tests")
    if not os.path.isdir(tests):
        pytest.skip("reference tests not copied (scripts/install_reference.sh)")
    files = [os.path.join(tests, t) for t in ("test_pipeline.py", "test_predict.py", "test_encode.py",
                                               "test_acceptance.py")]
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF, ROOT, tests]))
    p = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "paper_2509_20563_b200.plugin",
                        "-p", "no:cacheprovider", *files], cwd=tests, env=env, capture_output=True, text=True,
                       timeout=1800)
    tail = (p.stdout + p.stderr)[-4000:]
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "fzpipe_suite_with_plugin.log"), "w") as fh:
        fh.write(p.stdout + p.stderr)
    assert p.returncode == 0, tail
