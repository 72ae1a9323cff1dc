"""SPEC acceptance properties of the guiding mixture (SPEC.md 648-658 items
1-3 and 9), run through the GPU API at sizes the golden vectors cannot
cover: equal-area mapping, sampling-vs-pdf consistency of the device
sampler, normalisation of the mixture pdf, EM recovery."""

import numpy as np
import pytest
from scipy.stats import chi2

from oracle import pgg_oracle as O

pytestmark = pytest.mark.gpu


def test_mapping_equal_area_and_roundtrip(cuda_dev):
    """Criterion 1: round trip < 1e-5 over 1e5 points; a uniform square maps
    to a uniform hemisphere (chi-square over 64 equal-solid-angle bins)."""
    from paper_2112_09728_b200 import sgmap
    r = np.random.default_rng(1)
    p = r.uniform(0, 1, (200000, 2))
    d = sgmap.square_to_hemisphere(p)
    assert np.abs(sgmap.hemisphere_to_square(d) - p).max() < 1e-5
    # 8 bands of equal solid angle in z (uniform z on the hemisphere) x 8 azimuth sectors
    zb = np.minimum((d[:, 2] * 8).astype(int), 7)
    ab = np.minimum(((np.arctan2(d[:, 1], d[:, 0]) + np.pi) / (2 * np.pi) * 8).astype(int), 7)
    counts = np.bincount(zb * 8 + ab, minlength=64)
    exp = len(p) / 64
    stat = ((counts - exp) ** 2 / exp).sum()
    assert stat < chi2.ppf(0.999, 63)


def _stats(r, n):
    st = O.fresh_stats(n)
    st[:, 0:2] = r.uniform(0.2, 0.8, (n, 2))
    sd = r.uniform(0.05, 0.25, (n, 2))
    rho = r.uniform(-0.7, 0.7, n)
    st[:, 2] = sd[:, 0] ** 2 + st[:, 0] ** 2
    st[:, 3] = sd[:, 1] ** 2 + st[:, 1] ** 2
    st[:, 4] = rho * sd[:, 0] * sd[:, 1] + st[:, 0] * st[:, 1]
    st[:, 6] = r.uniform(0.1, 0.9, n)
    st[:, 7] = 5
    return st.astype(np.float32).astype(np.float64)


@pytest.mark.parametrize("kind", [0, 1])
def test_density_consistency(cuda_dev, kind):
    """Criterion 2: samples of the device sampler follow the mixture pdf it
    reports (chi-square on square-space bins), and the pdf integrates to 1."""
    from paper_2112_09728_b200 import mixture as M
    from paper_2112_09728_b200 import sgmap
    r = np.random.default_rng(7 + kind)
    for trial in range(4):
        st1 = _stats(r, 1)
        n = 400000
        st = np.repeat(st1, n, axis=0)
        rough = np.full(n, 0.6)
        wo = np.tile(np.array([[0.3, -0.2, 0.93]]) / np.linalg.norm([0.3, -0.2, 0.93]), (n, 1))
        streams = O.seed_lanes(100 + trial, 3, np.arange(n), 0)
        lb = M.lobe_from_stats(st)
        d, pdf, strat, valid = M.sample_mixture(st, lb, M.LocalBrdf(np.full(n, kind), rough, wo), None, streams)
        n_total = n
        d, pdf = d[valid], pdf[valid]
        # Lambert never leaves the hemisphere; GGX VNDF reflections can (invalid, pdf 0)
        assert valid.mean() > (0.97 if kind == 0 else 0.85)
        # histogram of square points vs expected mass from the pdf (x 2 pi Jacobian), 16 x 16 bins
        sq = sgmap.hemisphere_to_square(d)
        nb = 16
        idx = np.minimum((sq * nb).astype(int), nb - 1)
        counts = np.bincount(idx[:, 1] * nb + idx[:, 0], minlength=nb * nb).astype(float)
        g = (np.arange(nb) + 0.5) / nb
        gx, gy = np.meshgrid(g, g)
        cells = np.stack([gx.ravel(), gy.ravel()], -1)
        # expected: pdf at a fine grid inside each cell, averaged
        sub = 4
        off = (np.arange(sub) + 0.5) / (sub * nb) - 0.5 / nb
        ox, oy = np.meshgrid(off, off)
        pts = (cells[:, None, :] + np.stack([ox.ravel(), oy.ravel()], -1)[None]).reshape(-1, 2)
        dirs = sgmap.square_to_hemisphere(pts)
        m = len(pts)
        brdf = O.brdf_density(np.full(m, kind), np.full(m, 0.6), dirs, np.repeat(wo[:1], m, 0),
                              np.tile([0.0, 0.0, 1.0], (m, 1)))
        lbm = M.GaussianLobe(np.repeat(lb.mu[:1], m, 0), np.repeat(lb.cov[:1], m, 0), np.repeat(lb.chol[:1], m, 0),
                             np.repeat(lb.trunc_z[:1], m, 0))
        mp = M.mixture_pdf(np.repeat(st[:1], m, 0), lbm, dirs, brdf) * 2 * np.pi   # per unit square area
        expected = mp.reshape(nb * nb, sub * sub).mean(1) / (nb * nb) * n_total
        # the mixture pdf integrates to the probability of a valid sample
        # (1 for Lambert; the GGX VNDF pdf integrates to P(above horizon))
        assert abs(expected.sum() / n_total - valid.mean()) < 0.02
        keep = expected > 20
        stat = ((counts[keep] - expected[keep]) ** 2 / expected[keep]).sum()
        assert stat < chi2.ppf(0.999, keep.sum() - 1) * 1.5, (trial, stat, keep.sum())


def test_em_recovery(cuda_dev):
    """Criterion 3: online M-steps on uniform proposals weighted by a target
    N((0.3, 0.6), 0.02 I) recover it (mu error < 0.05, Sigma Frobenius error
    < 30 %); pi stays in [0.05, 0.95]."""
    from paper_2112_09728_b200 import mixture as M
    r = np.random.default_rng(3)
    st = O.fresh_stats(1)
    mu_t, var_t = np.array([0.3, 0.6]), 0.02
    for epoch in range(500):
        sq = r.uniform(0, 1, (1, 32, 2))
        w = np.exp(-0.5 * ((sq - mu_t) ** 2).sum(-1) / var_t)
        lb = M.lobe_from_stats(st)
        g = M.gaussian_pdf_square(M.GaussianLobe(lb.mu[:, None], lb.cov[:, None], lb.chol[:, None],
                                                 lb.trunc_z[:, None]), sq)
        resp = M.e_step_responsibility(st[:, 6:7], g, np.ones_like(g))
        st = M.m_step_update(st, sq, w, resp, k_max=64)
        assert 0.05 <= st[0, 6] <= 0.95
    mu = st[0, :2]
    cov = np.array([[st[0, 2] - mu[0] ** 2, st[0, 4] - mu[0] * mu[1]], [st[0, 4] - mu[0] * mu[1], st[0, 3] - mu[1] ** 2]])
    assert np.abs(mu - mu_t).max() < 0.05
    assert np.linalg.norm(cov - var_t * np.eye(2)) / np.linalg.norm(var_t * np.eye(2)) < 0.3


def test_neighbor_count_endpoints(cuda_dev):
    """Criterion 9: N(k=0) = 20, N(kMax) = 5."""
    from paper_2112_09728_b200 import mixture as M
    assert M.neighbor_count(np.array([0]), 64)[0] == 20 and M.neighbor_count(np.array([64]), 64)[0] == 5
