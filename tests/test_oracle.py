"""Pin the CPU oracle (oracle/pgg_oracle.py) against the reference's own
outputs (tests/golden/*.npz) and the SPEC known-answer examples
(SURVEY.md section 4).  CPU only."""

import numpy as np
import pytest

import golden_io as gio
from oracle import pgg_oracle as O


@pytest.fixture(scope="module")
def kat():
    return gio.load("kat.npz")


@pytest.fixture(scope="module")
def seq():
    return gio.load("seq_64x48.npz")


@pytest.fixture(scope="module")
def trained():
    return gio.load("trained_48x40.npz")


def test_pcg_vectors(kat):
    s = O.seed_lanes(0, 0, np.arange(4))
    assert O.draw_u32(s).tolist() == [1205138062, 2492159297, 3840735293, 3518835114]
    assert O.draw_u32(s).tolist() == [2755668754, 1954364939, 1526284107, 473607138]
    np.testing.assert_array_equal(kat["pcg_0_0_a"], [1205138062, 2492159297, 3840735293, 3518835114])
    s = O.seed_lanes(3, 1, np.array([0, 1]), stream=1)
    assert O.draw_u32(s).tolist() == [3445375490, 1865877714] == kat["pcg_3_1_s1"].tolist()
    s = O.seed_lanes(123456789, 77, np.arange(1000, 1064) * 7, 0)
    np.testing.assert_array_equal(s, kat["pcg_big_state0"])
    np.testing.assert_array_equal(np.stack([O.draw_u32(s) for _ in range(40)]), kat["pcg_big"])


def test_sgmap_kat(kat):
    np.testing.assert_allclose(O.sq_to_dir([0.5, 0.5]), [0, 0, 1], atol=0)
    np.testing.assert_allclose(O.sq_to_dir([1.0, 0.5]), [1, 0, 0], atol=1e-15)
    d = O.sq_to_dir(kat["sg_sq"])
    np.testing.assert_array_equal(d, kat["sg_dir"])
    np.testing.assert_array_equal(O.dir_to_sq(d), kat["sg_back"])
    assert np.abs(kat["sg_back"] - kat["sg_sq"]).max() < 1e-12
    with pytest.raises(ValueError):
        O.dir_to_sq([0.0, 0.0, -0.5])
    assert abs(1.0 / (2 * np.pi) - 0.15915494) < 1e-8
    t, b = O.onb(kat["onb_n"])
    np.testing.assert_array_equal(t, kat["onb_t"])
    np.testing.assert_array_equal(b, kat["onb_b"])


def test_lobe_and_trunc(kat):
    lb = O.lobe(kat["lobe_stats"].astype(np.float64))
    np.testing.assert_array_equal(lb.mu, kat["lobe_mu"])
    np.testing.assert_array_equal(lb.cov, kat["lobe_cov"])
    np.testing.assert_array_equal(lb.chol, kat["lobe_chol"])
    np.testing.assert_allclose(lb.z, kat["lobe_z"], rtol=1e-13)
    np.testing.assert_allclose(O.gauss_sq_pdf(lb, kat["lobe_qp"]), kat["lobe_pdf"], rtol=1e-13)
    # SPEC KATs (code wins over SPEC prose): init -> Sigma = 0.2501 I, no reset
    init = O.lobe(O.fresh_stats(1))
    assert not init.reset[0]
    np.testing.assert_allclose(init.cov[0], [[0.2501, 0], [0, 0.2501]], rtol=1e-14)
    # m2 = mu mu^T -> ridge keeps lambda_min = 1e-4 > 1e-6: no reset, cov = 1e-4 I
    st = O.fresh_stats(1)
    st[0, O.M2_XX], st[0, O.M2_YY], st[0, O.M2_XY] = 0.25, 0.25, 0.25
    lb = O.lobe(st)
    assert not lb.reset[0]
    np.testing.assert_allclose(lb.cov[0], 1e-4 * np.eye(2), atol=1e-18)
    # indefinite -> reset to 0.05 I
    st[0, O.M2_XY] = 0.6
    assert O.lobe(st).reset[0]
    # truncation-mass clamp and symmetric cases
    z = O.trunc_mass(np.array([5.0]), np.array([5.0]), np.array([0.01]), np.array([0.0]), np.array([0.01]))
    assert z[0] == 1e-4
    z = O.trunc_mass(np.array([0.5]), np.array([0.5]), np.array([0.01]), np.array([0.0]), np.array([0.01]))
    assert abs(z[0] - 1.0) < 1e-6  # GL24 over +-8.5 sigma: 6.1e-7 short
    z = O.trunc_mass(np.array([0.0]), np.array([0.5]), np.array([0.01]), np.array([0.0]), np.array([0.01]))
    assert abs(z[0] - 0.5) < 1e-6


def test_mstep_estep_budget(kat):
    out = O.m_step(kat["ms_stats"], kat["ms_sq"], kat["ms_w"], kat["ms_r"], kat["ms_valid"], 64)
    np.testing.assert_allclose(out, kat["ms_out"], rtol=1e-14, atol=1e-300)
    np.testing.assert_array_equal(O.budget(kat["nc_k"], 64), kat["nc_n"])
    assert O.budget(0, 64) == 20 and O.budget(64, 64) == 5 and O.budget(32, 64) == 13
    # SPEC E-step examples
    assert O.responsibility(0.5, 1.0, 1.0) == 0.5
    assert O.responsibility(0.5, 1.0, 0.0) == 1.0
    assert abs(O.responsibility(0.4, 1.0, 1.0) - 0.4) < 1e-15
    assert O.responsibility(0.5, 0.0, 0.0) == 0.0
    # SPEC M-step k=0 single sample (0.3, 0.7)
    st = O.fresh_stats(1)
    o = O.m_step(st, np.array([[[0.3, 0.7]]]), np.array([[1.0]]), np.array([[1.0]]), np.array([[True]]), 64)
    np.testing.assert_allclose(o[0], [0.3, 0.7, 0.09, 0.49, 0.21, 1.0, 0.95, 1.0], rtol=1e-14)
    # empty batch -> unchanged
    o = O.m_step(st, np.zeros((1, 0, 2)), np.zeros((1, 0)), np.zeros((1, 0)), np.zeros((1, 0), bool), 64)
    np.testing.assert_array_equal(o, st)
    bm = O.box_muller(kat["bm_u"][0], kat["bm_u"][1])
    np.testing.assert_array_equal(np.stack(bm), kat["bm_out"])
    np.testing.assert_allclose(O.box_muller(0.5, 0.5), (-1.1774100225154747, 0), atol=1e-12)


@pytest.mark.parametrize("frame", range(6))
def test_sequence_frame(seq, frame):
    """Each stage of each frame, fed the reference's own inputs."""
    z, f = seq, frame
    spp, seed = int(z["spp"]), int(z["seed"])
    g = gio.gbuf(z, f"f{f}_")
    v = gio.vpl(z, f"f{f}_")
    if f > 0:
        gp = gio.gbuf(z, f"f{f-1}_")
        rep = O.reproject(z[f"f{f}_gamma_in"], gp, g)
        np.testing.assert_array_equal(rep, z[f"f{f}_gamma_reproj"])
    gam = z[f"f{f}_gamma_reproj"]
    smp = O.sample_frame(gam, g, seed, f, spp=spp, nee_draws=3)
    np.testing.assert_array_equal(smp["valid"], z[f"f{f}_smp_valid"])
    np.testing.assert_array_equal(smp["strategy"], z[f"f{f}_smp_strategy"])
    np.testing.assert_allclose(smp["wi"], z[f"f{f}_smp_wi"], rtol=0, atol=1e-14)
    np.testing.assert_allclose(smp["pdf"], z[f"f{f}_smp_pdf"], rtol=1e-12)
    tr = O.train(gam, v, g, 64, seed, f)
    d = gio.ulp_diff_f32(tr, z[f"f{f}_gamma_trained"])
    assert d.max() <= 1, d.max()


def test_trained_frame(trained):
    z = trained
    spp, seed, fr = int(z["spp"]), int(z["seed"]), int(z["frame"])
    gp, g = gio.gbuf(z, "p_"), gio.gbuf(z, "c_")
    v = gio.vpl(z, "c_")
    np.testing.assert_array_equal(O.reproject(z["gamma_in"], gp, g), z["gamma_reproj"])
    smp = O.sample_frame(z["gamma_in"], g, seed, fr, spp=spp, nee_draws=3)
    np.testing.assert_array_equal(smp["valid"], z["smp_valid"])
    np.testing.assert_array_equal(smp["strategy"], z["smp_strategy"])
    np.testing.assert_allclose(smp["wi"], z["smp_wi"], rtol=0, atol=1e-14)
    np.testing.assert_allclose(smp["pdf"], z["smp_pdf"], rtol=1e-12)
    tr = O.train(z["gamma_in"], v, g, 64, seed, fr)
    assert gio.ulp_diff_f32(tr, z["gamma_trained"]).max() <= 1
    tr = O.train(z["gamma_in"], v, g, 32, seed, fr, radius=7.3)
    assert gio.ulp_diff_f32(tr, z["gamma_trained_r7"]).max() <= 1


@pytest.mark.parametrize("rows", [(0, 11), (11, 30), (30, 40)])
def test_row_band_equals_whole_frame(trained, rows):
    """The oracle's row-band mode (whole frame as context, global stream
    keys) reproduces the same rows of the whole-frame oracle bit for bit --
    which is what lets the 1080p parity test check full-width bands, frame
    edges included, without running the oracle on the whole frame."""
    z = trained
    spp, seed, fr = int(z["spp"]), int(z["seed"]), int(z["frame"])
    gp, g = gio.gbuf(z, "p_"), gio.gbuf(z, "c_")
    v = gio.vpl(z, "c_")
    rep, smp, tr = O.guiding_frame(z["gamma_in"], gp, g, v, seed, fr, spp=spp)
    rep_b, smp_b, tr_b = O.guiding_frame(z["gamma_in"], gp, g, v, seed, fr, spp=spp, rows=rows)
    r0, r1 = rows
    w = g.valid.shape[1]
    np.testing.assert_array_equal(rep_b, rep[r0:r1])
    np.testing.assert_array_equal(tr_b, tr[r0:r1])
    for k in ("wi", "pdf", "strategy", "valid", "draws"):
        np.testing.assert_array_equal(smp_b[k], smp[k][r0 * w:r1 * w])
