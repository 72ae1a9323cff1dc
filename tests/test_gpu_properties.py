"""Property-based parity (hypothesis) of the GPU lane APIs against the
oracle on arbitrary, adversarial inputs: lobe / truncation mass on random
moment sets (tight, correlated, indefinite, boundary means), the M-step on
random batches with invalid and non-finite records, and PCG stream jumps."""

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from oracle import pgg_oracle as O

pytestmark = pytest.mark.gpu

floats01 = st.floats(0.0, 1.0, allow_nan=False)


def _stats(mx, my, sx, sy, rho, pi, k):
    s = np.array([[mx, my, sx * sx + mx * mx, sy * sy + my * my, rho * sx * sy + mx * my, 0.0, pi, k]])
    return s.astype(np.float32).astype(np.float64)


@settings(max_examples=60, deadline=None, suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(mx=floats01, my=floats01, sx=st.floats(1e-4, 0.6), sy=st.floats(1e-4, 0.6), rho=st.floats(-0.999, 0.999),
       pi=st.floats(0.05, 0.95), k=st.integers(0, 200))
def test_lobe_matches_oracle(cuda_dev, mx, my, sx, sy, rho, pi, k):
    from paper_2112_09728_b200 import mixture as M
    s = _stats(mx, my, sx, sy, rho, pi, k)
    lb = M.lobe_from_stats(s)
    ref = O.lobe(s)
    np.testing.assert_array_equal(lb.mu, ref.mu)               # float64, reference operation order
    np.testing.assert_allclose(lb.chol[0, 0, 0], ref.l11, rtol=1e-15)
    np.testing.assert_allclose(lb.chol[0, 1, 1], ref.l22, rtol=1e-15)
    # truncation mass: exact BVN vs the reference's 5 x 24 Gauss-Legendre rule
    assert abs(lb.trunc_z[0] - ref.z[0]) <= 1e-4 * max(ref.z[0], 1e-4) + 2e-6


@settings(max_examples=40, deadline=None, suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(seed=st.integers(0, 2**31 - 1), n=st.integers(1, 20), k=st.integers(0, 100), kmax=st.integers(1, 80),
       bad=st.floats(0.0, 0.5))
def test_m_step_matches_oracle(cuda_dev, seed, n, k, kmax, bad):
    from paper_2112_09728_b200 import mixture as M
    r = np.random.default_rng(seed)
    s = _stats(r.uniform(), r.uniform(), r.uniform(0.01, 0.3), r.uniform(0.01, 0.3), r.uniform(-0.9, 0.9),
               r.uniform(0.05, 0.95), k)
    sq = r.uniform(0, 1, (1, n, 2))
    w = r.exponential(1.0, (1, n))
    resp = r.uniform(0, 1, (1, n))
    valid = r.uniform(0, 1, (1, n)) > bad
    w[0, r.uniform(0, 1, n) < bad / 4] = np.nan  # non-finite weights are dropped
    got = M.m_step_update(s, sq, w, resp, valid=valid, k_max=kmax)
    ok = valid & np.isfinite(w) & (w >= 0)
    ref = O.m_step(s, sq, np.where(ok, w, 0.0), resp, ok, kmax)
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-300)


@settings(max_examples=30, deadline=None, suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(seed=st.integers(0, 2**63 - 1), frame=st.integers(0, 2**32), lanes=st.lists(st.integers(0, 2**40), min_size=1,
                                                                                   max_size=16))
def test_streams_match_oracle(cuda_dev, seed, frame, lanes):
    from paper_2112_09728_b200 import rng
    s = rng.make_streams(seed, frame, np.array(lanes, dtype=np.uint64))
    ref = O.seed_lanes(seed, frame, np.array(lanes, dtype=np.uint64), 0)
    np.testing.assert_array_equal(s, ref)
    for _ in range(5):
        np.testing.assert_array_equal(rng.next_u32(s), O.draw_u32(ref))
