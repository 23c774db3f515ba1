"""1D Lorenzo fields read once before their bound (fzb_lorenzo1d_prepare_f32):
the walker's summary pass also yields the field's (min, max) and the
non-finite check of fzb_minmax_f32 (pipeline.py:360-361).  The archive
header's lo / hi and every archive byte must equal the oracle's; NaN / inf
anywhere (including the partial last 1024-element block) must raise like
the min/max pass; a signed-zero minimum keeps its sign."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2509_20563_b200 as fz  # noqa: E402
from paper_2509_20563_b200.data import particle1d_host  # noqa: E402

EB = fz.ErrorBoundSpec(fz.ErrorMode.VALUE_RANGE_RELATIVE, 1e-4)


@pytest.mark.parametrize("n", [1, 31, 1024, 1025, 40000, 1 << 20, (1 << 20) + 777])
@pytest.mark.parametrize("preset", ["default", "speed"])
def test_1d_archive_matches_oracle(oracle, n, preset):
    x = particle1d_host(n, n)
    blob = fz.serialize_archive(fz.compress(fz.Field((n,), x), EB, preset))
    assert blob == oracle.compress(x, (n,), 1, 1e-4, preset)


@pytest.mark.parametrize("n,where", [(5000, 0), (5000, 4999), (5000, 2500), (1 << 16, (1 << 16) - 1), (1025, 1024)])
@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_1d_nonfinite_raises(n, where, bad):
    x = particle1d_host(n, 3).copy()
    x[where] = bad
    with pytest.raises(ValueError, match="non-finite"):
        fz.compress(fz.Field((n,), x), EB, "default")


@pytest.mark.parametrize("dims", [(4096,), (16, 16, 16)])
@pytest.mark.parametrize("zero", [-0.0, 0.0])
def test_signed_zero_minimum_matches_oracle(oracle, dims, zero):
    # the minimum is a zero of one sign: deterministic for numpy and the GPU.
    # (Both signs at once: numpy's min returns either, depending on its SIMD
    # reduction order -- see DESIGN.md section 2; only the header's lo differs.)
    n = int(np.prod(dims))
    rng = np.random.default_rng(9)
    x = rng.uniform(0.0, 1.0, n).astype(np.float32)
    x[rng.choice(n, 20, replace=False)] = np.float32(zero)
    blob = fz.serialize_archive(fz.compress(fz.Field(dims, x.reshape(dims)), EB, "default"))
    assert blob == oracle.compress(x, dims, 1, 1e-4, "default")
