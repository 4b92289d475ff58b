"""GPU: the device-side generator (rsm_ctx_generate)
against the host generator rsm_generate (itself pinned to the oracle's
restatement of src/synth.cpp:12-57 in test_gpu_parity): the mask bit-exactly,
the values to a few ulps (Box-Muller's log/cos come from the device math
library, not glibc), and the decomposition of the two inputs to the
north-star tolerance with equal report fields."""
import numpy as np
import pytest

from paper_1411_0814_b200 import rsm
from tests.util import rel_fro

pytestmark = pytest.mark.gpu

VAL_TOL = 1e-13  # |y_dev - y_host| <= VAL_TOL * max(1, |y_host|): a few ulps of the factor sums


def _compare(m, n, r, rho, sigma, seed):
    ctx = rsm.Context(0)
    ctx.generate(m, n, r, rho, sigma, seed)
    D = ctx.fetch_matrix()
    H = rsm.generate(m, n, r, rho, sigma, seed)
    assert np.array_equal(D.mask, H.mask), "mask must be bit-exact"
    hid = H.mask == 0
    assert np.isnan(D.values[hid]).all()
    dv, hv = D.values[~hid], H.values[~hid]
    err = np.abs(dv - hv) / np.maximum(1.0, np.abs(hv))
    assert err.max() <= VAL_TOL, f"max scaled value difference {err.max():.3e}"
    return ctx, D, H, float(np.mean(dv == hv))


@pytest.mark.parametrize("shape", [(300, 77, 3, 0.8, 1e-3, 0), (257, 130, 5, 0.7, 1e-2, 3), (64, 33, 1, 1.0, 0.0, 9)])
def test_device_generator_matches_host(shape):
    _, _, _, same = _compare(*shape)
    assert same > 0.5  # most values are bit-identical; the rest differ in the last ulps


def test_device_generator_config3_full_size():
    # BASELINE config 3 at full size: 131072 x 1024, r = 4, rho = 0.8
    _, D, H, same = _compare(131072, 1024, 4, 0.8, 1e-3, 0)
    assert abs(D.mask.mean() - 0.8) < 1e-3


def test_decompose_on_device_generated_input():
    m, n, r = 2000, 200, 3
    ctx, D, H, _ = _compare(m, n, r, 0.8, 1e-3, 0)
    cfg = rsm.RsmConfig(rank=r, mode=rsm.Mode.M2, block=4, plan=rsm.TrialPlan(2000), seed=0)
    Fd, repd = ctx.decompose(cfg)
    Fh, reph = rsm.decompose(H, cfg)
    assert (repd.trials_attempted, repd.trials_accepted, repd.z, repd.gram_rank, repd.underdetermined_rows) == (
        reph.trials_attempted, reph.trials_accepted, reph.z, reph.gram_rank, reph.underdetermined_rows)
    assert rel_fro(Fd.u @ Fd.v.T, Fh.u @ Fh.v.T) <= 1e-9
    assert abs(repd.e - reph.e) <= 1e-9 * reph.e


def test_device_generator_validation():
    ctx = rsm.Context(0)
    for bad in [(0, 10, 2, 0.5, 0.0, 0), (10, 10, 0, 0.5, 0.0, 0), (10, 10, 2, 0.0, 0.0, 0), (10, 10, 2, 0.5, -1.0, 0)]:
        with pytest.raises(rsm.Error) as ei:
            ctx.generate(*bad)
        assert ei.value.code == rsm.errc.invalid_config
