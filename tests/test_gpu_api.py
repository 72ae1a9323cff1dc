"""The reference-compatible Python API (paper_2112_09728_b200.{rng, mixture,
sgmap, ptrace, guide_buffers}) on the GPU against the reference golden
vectors and the oracle, called the way pgtrace callers call pgtrace."""

from types import SimpleNamespace

import numpy as np
import pytest

import golden_io as gio
from oracle import pgg_oracle as O
from test_hostcheck import check_gamma, check_samples

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kat():
    return gio.load("kat.npz")


def test_rng_api(cuda_dev, kat):
    from paper_2112_09728_b200 import rng
    s = rng.make_streams(0, 0, np.arange(4))
    assert s.dtype == np.uint64
    assert rng.next_u32(s).tolist() == [1205138062, 2492159297, 3840735293, 3518835114]
    assert rng.next_u32(s).tolist() == [2755668754, 1954364939, 1526284107, 473607138]   # in place
    s = rng.make_streams(3, 1, np.array([0, 1]), stream_id=1)
    assert rng.next_u32(s).tolist() == [3445375490, 1865877714]
    s = rng.make_streams(123456789, 77, np.arange(1000, 1064) * 7, stream_id=0)
    np.testing.assert_array_equal(s, kat["pcg_big_state0"])
    np.testing.assert_array_equal(np.stack([rng.next_u32(s) for _ in range(40)]), kat["pcg_big"])
    s2 = O.seed_lanes(5, 6, np.arange(100), 1)
    s1 = rng.make_streams(5, 6, np.arange(100), 1)
    np.testing.assert_array_equal(rng.next_f64(s1), O.draw_unit(s2))
    np.testing.assert_array_equal(s1, s2)


def test_mixture_api(cuda_dev, kat):
    from paper_2112_09728_b200 import mixture as M
    st = kat["lobe_stats"].astype(np.float64)
    lb = M.lobe_from_stats(st)
    np.testing.assert_array_equal(lb.mu, kat["lobe_mu"])
    np.testing.assert_array_equal(lb.cov, kat["lobe_cov"])
    np.testing.assert_array_equal(lb.chol, kat["lobe_chol"])
    # the API evaluates the reference's own rule in float64 (the pass uses its
    # float32 Genz form, test_hostcheck.test_lobe_trunc_mass / tools/trunc_fuzz.py)
    assert gio.rel_err(lb.trunc_z, kat["lobe_z"]).max() <= 1e-12
    np.testing.assert_allclose(M.truncation_mass(kat["lobe_mu"], kat["lobe_cov"]), lb.trunc_z, rtol=0, atol=0)
    ref_lobe = O.lobe(st)
    ref_pdf = O.gauss_sq_pdf(SimpleNamespace(mu=ref_lobe.mu, l11=ref_lobe.l11, l21=ref_lobe.l21, l22=ref_lobe.l22,
                                             z=kat["lobe_z"]), kat["lobe_qp"])
    pdf = M.gaussian_pdf_square(M.GaussianLobe(lb.mu, lb.cov, lb.chol, kat["lobe_z"]), kat["lobe_qp"])
    np.testing.assert_allclose(pdf, ref_pdf, rtol=1e-12)
    out = M.m_step_update(kat["ms_stats"], kat["ms_sq"], kat["ms_w"], kat["ms_r"], valid=kat["ms_valid"], k_max=64)
    np.testing.assert_allclose(out, kat["ms_out"], rtol=1e-12, atol=1e-300)
    np.testing.assert_array_equal(M.neighbor_count(kat["nc_k"], 64), kat["nc_n"])
    bm = M.box_muller(kat["bm_u"][0], kat["bm_u"][1])
    np.testing.assert_allclose(np.stack(bm), kat["bm_out"], rtol=1e-13, atol=1e-13)
    assert M.e_step_responsibility(0.5, 1.0, 1.0) == 0.5 and M.e_step_responsibility(0.5, 0.0, 0.0) == 0.0
    np.testing.assert_array_equal(M.init_stats((2, 3))[1, 2], [0.5, 0.5, 0.5, 0.5, 0.25, 0.0, 0.05, 0.0])


def test_sample_mixture_api(cuda_dev):
    """Local-frame mixture draws == oracle: strategies, validity and final
    stream states bitwise; directions / pdfs within policy."""
    from paper_2112_09728_b200 import mixture as M
    r = np.random.default_rng(4)
    n = 20000
    st = O.fresh_stats(n)
    st[:, 0:2] = r.uniform(0.1, 0.9, (n, 2))
    sd = 10 ** r.uniform(-1.5, -0.5, (n, 2))
    rho = r.uniform(-0.8, 0.8, n)
    st[:, 2] = sd[:, 0] ** 2 + st[:, 0] ** 2
    st[:, 3] = sd[:, 1] ** 2 + st[:, 1] ** 2
    st[:, 4] = rho * sd[:, 0] * sd[:, 1] + st[:, 0] * st[:, 1]
    st[:, 6] = r.uniform(0.05, 0.95, n)
    st = st.astype(np.float32).astype(np.float64)
    kind = (r.uniform(0, 1, n) < 0.4).astype(np.int64)
    rough = r.uniform(0.05, 1.0, n).astype(np.float32).astype(np.float64)
    wo = r.normal(size=(n, 3))
    wo[:, 2] = np.abs(wo[:, 2]) + 0.05
    wo = (wo / np.linalg.norm(wo, axis=1, keepdims=True)).astype(np.float32).astype(np.float64)
    streams = O.seed_lanes(9, 1, np.arange(n), 0)
    ref_states = streams.copy()
    lb = M.lobe_from_stats(st)
    d, pdf, strat, valid = M.sample_mixture(st, lb, M.LocalBrdf(kind, rough, wo), None, streams)
    olb = O.lobe(st)
    olb.z = lb.trunc_z
    od, opdf, ostrat, ovalid = O.draw_mixture(st, olb, kind, rough, wo, ref_states)
    np.testing.assert_array_equal(streams, ref_states)
    np.testing.assert_array_equal(strat, ostrat)
    np.testing.assert_array_equal(valid, ovalid)
    assert np.abs(d - od).max() <= 1e-5
    rr = gio.rel_err(pdf, opdf)
    assert np.percentile(rr, 99.99) <= 1e-4 and rr.max() <= 1e-3
    # the reference's callback form (pg/mixture.py:193-205, pg/ptrace.py:201-208):
    # Gaussian branch on the device, the caller's BRDF sampler / pdf on the host
    ez = np.broadcast_to(np.array([0.0, 0.0, 1.0]), (n, 3))
    calls = []

    def cb_sample(rel, sub):
        calls.append(("sample", rel.copy()))
        w_l, _, ok = O.brdf_draw(kind[rel], rough[rel], wo[rel], ez[rel], sub)
        return w_l, ok

    def cb_pdf(rel, dirs_l):
        calls.append(("pdf", rel.copy()))
        return O.brdf_density(kind[rel], rough[rel], dirs_l, wo[rel], ez[rel])

    streams = O.seed_lanes(9, 1, np.arange(n), 0)
    ref_states = streams.copy()
    d, pdf, strat, valid = M.sample_mixture(st, lb, cb_sample, cb_pdf, streams)
    od, opdf, ostrat, ovalid = O.draw_mixture(st, olb, kind, rough, wo, ref_states)
    np.testing.assert_array_equal(streams, ref_states)
    np.testing.assert_array_equal(strat, ostrat)
    np.testing.assert_array_equal(valid, ovalid)
    np.testing.assert_allclose(d, od, rtol=0, atol=1e-12)
    np.testing.assert_allclose(pdf, opdf, rtol=1e-10, atol=0)
    assert [c[0] for c in calls] == ["sample", "pdf"]
    np.testing.assert_array_equal(calls[0][1], np.nonzero(ostrat == 0)[0])  # exactly the reference's lanes


def _ref_gbuf(z, prefix):
    g = gio.gbuf(z, prefix)
    return g


def test_guide_buffers_api_golden(cuda_dev):
    from paper_2112_09728_b200 import guide_buffers as GB
    from paper_2112_09728_b200 import ptrace as PT
    z = gio.load("seq_64x48.npz")
    seed, spp = int(z["seed"]), int(z["spp"])
    for f in (1, 4):
        g, gp, v = gio.gbuf(z, f"f{f}_"), gio.gbuf(z, f"f{f-1}_"), gio.vpl(z, f"f{f}_")
        gam = GB.GuidingBuffer(64, 48, z[f"f{f}_gamma_in"], generation=3)
        rep = GB.reproject(gam, gp, g, GB.ReprojectionPolicy())
        assert isinstance(rep.stats, np.ndarray) and rep.stats.dtype == np.float32 and rep.generation == 4
        check_gamma(rep.stats, z[f"f{f}_gamma_reproj"])
        tr = GB.training_pass(GB.GuidingBuffer(64, 48, z[f"f{f}_gamma_reproj"]), v, g, k_max=64, seed=seed,
                              frame_index=f)
        check_gamma(tr.stats, z[f"f{f}_gamma_trained"])
        smp = PT.sample_first_bounce_frame(z[f"f{f}_gamma_reproj"], g, seed, f, spp=spp)
        check_samples(smp, z[f"f{f}_smp_wi"], z[f"f{f}_smp_pdf"], z[f"f{f}_smp_strategy"], z[f"f{f}_smp_valid"])
        g_rep, smp2, g_tr = GB.guiding_frame(gam, gp, g, v, seed=seed, frame_index=f, spp=spp)
        check_gamma(g_rep.stats, z[f"f{f}_gamma_reproj"])


def test_first_bounce_api_golden(cuda_dev):
    """ptrace._sample_first_bounce on the golden lanes, streams in/out."""
    from paper_2112_09728_b200 import mixture as M
    from paper_2112_09728_b200 import ptrace as PT
    from paper_2112_09728_b200 import synth
    z = gio.load("seq_64x48.npz")
    seed, spp, f = int(z["seed"]), int(z["spp"]), 3
    g = gio.gbuf(z, f"f{f}_")
    kind, rough, alb = synth._materials(seed, "cpu")
    scene = SimpleNamespace(mat_kind=kind.numpy().astype(np.int64), mat_rough=rough.numpy().astype(np.float64),
                            mat_albedo=alb.numpy().astype(np.float64))
    stats = z[f"f{f}_gamma_reproj"].reshape(-1, 8).astype(np.float64)
    valid = g.valid.reshape(-1)
    pix = np.nonzero(valid)[0]
    lob = M.lobe_from_stats(stats[pix])
    guided = valid[pix] & ((g.kind.reshape(-1)[pix] == 0) | (g.roughness.reshape(-1)[pix] >= 0.05)) & (
        stats[pix, 7] >= 1.0)
    s = 1
    streams = O.seed_lanes(seed, f, pix.astype(np.uint64) * np.uint64(spp) + np.uint64(s), 0)
    for _ in range(3):
        O.draw_u32(streams)
    wi, pdf, strat, ok = PT._sample_first_bounce(scene, np.arange(pix.size), g.pos.reshape(-1, 3)[pix],
                                                 g.normal.reshape(-1, 3)[pix], np.maximum(g.mat.reshape(-1)[pix], 0),
                                                 g.view.reshape(-1, 3)[pix], stats[pix], lob, guided, streams)
    np.testing.assert_array_equal(streams, z[f"f{f}_smp_state"][pix, s])
    np.testing.assert_array_equal(strat, z[f"f{f}_smp_strategy"][pix, s])
    np.testing.assert_array_equal(ok, z[f"f{f}_smp_valid"][pix, s])
    assert np.abs(wi - z[f"f{f}_smp_wi"][pix, s]).max() <= 1e-5


def test_gather_training_batch_api(cuda_dev):
    from paper_2112_09728_b200 import guide_buffers as GB
    z = gio.load("trained_48x40.npz")
    g, v = gio.gbuf(z, "c_"), gio.vpl(z, "c_")
    gam = GB.GuidingBuffer(48, 40, z["gamma_in"])
    for (x, y) in ((5, 7), (20, 30), (0, 0), (47, 39)):
        st_g = O.seed_lanes(2, 3, np.arange(48 * 40), 1)
        st_o = st_g.copy()
        recs = GB.gather_training_batch((x, y), v, g, gam, 64, st_g)
        # oracle: records of that pixel from the same streams
        stats = z["gamma_in"].reshape(-1, 8).astype(np.float64)
        cand, used = O.candidates(40, 48, 10.0, st_o)
        used &= np.arange(20)[None, :] < O.budget(stats[:, 7], 64)[:, None]
        sq, w, r, ok = O.records(stats, O.lobe(stats), v, g, cand, used)
        np.testing.assert_array_equal(st_g, st_o)   # both advanced by the 38 draws
        p = y * 48 + x
        assert len(recs) == int(ok[p].sum())
        slots = np.nonzero(ok[p])[0]
        for rec, s in zip(recs, slots):
            assert np.abs(rec.sq - sq[p, s]).max() <= 1e-5
            assert abs(rec.weight - w[p, s]) <= 1e-4 * max(abs(w[p, s]), 1e-7)


def test_checkpoint_roundtrip(tmp_path, cuda_dev):
    from paper_2112_09728_b200 import guide_buffers as GB
    g = GB.GuidingBuffer.create(17, 9)
    g.stats[3, 4, 0] = 0.123
    p = tmp_path / "g.pgg"
    GB.checkpoint_save(g, p)
    h = GB.checkpoint_load(p, expect_size=(17, 9))
    np.testing.assert_array_equal(h.stats, g.stats)
    with pytest.raises(GB.CheckpointError):
        GB.checkpoint_load(p, expect_size=(9, 17))


def test_sgmap_lane_kernels(cuda_dev, kat):
    """sgmap (pgg_sgmap lane kernels) vs the oracle's float64 restatement and
    the reference's round-trip KATs."""
    import torch

    from paper_2112_09728_b200 import sgmap
    r = np.random.default_rng(12)
    p = r.uniform(0, 1, (50000, 2))
    p[:4] = [[0.5, 0.5], [0.0, 0.0], [1.0, 0.5], [0.5, 1.0]]
    d = sgmap.square_to_hemisphere(p)
    np.testing.assert_allclose(d, O.sq_to_dir(p), rtol=0, atol=1e-15)
    v = d / np.linalg.norm(d, axis=-1, keepdims=True)
    np.testing.assert_allclose(sgmap.hemisphere_to_square(v), O.dir_to_sq(v), rtol=0, atol=1e-14)
    disk = sgmap.square_to_disk(p)
    np.testing.assert_allclose(sgmap.disk_to_square(disk), p, rtol=0, atol=1e-14)
    n = r.standard_normal((1000, 3))
    n /= np.linalg.norm(n, axis=-1, keepdims=True)
    t, b = sgmap.build_tangent_frame(n)
    ot, ob = O.onb(n)
    np.testing.assert_array_equal(t, ot)
    np.testing.assert_array_equal(b, ob)
    loc = r.standard_normal((1000, 3))
    np.testing.assert_allclose(sgmap.to_world(t, b, n, loc), O.local_to_world(ot, ob, n, loc), rtol=0, atol=1e-15)
    np.testing.assert_allclose(sgmap.to_local(t, b, n, loc), O.world_to_local(ot, ob, n, loc), rtol=0, atol=1e-15)
    assert sgmap.square_density_to_solid_angle(2 * np.pi) == 1.0
    with pytest.raises(ValueError):
        sgmap.hemisphere_to_square(np.array([[0.0, 0.0, -1.0]]))
    tp = torch.as_tensor(p[:10], device=cuda_dev)
    assert torch.is_tensor(sgmap.square_to_hemisphere(tp))


def test_pack_gbuffer_mat_equals_pack(cuda_dev):
    """pgg_pack_gbuffer_mat (material ids + the scene's material table, the
    lookups of pg/ptrace.py:97-129) builds the same planes, bit for bit, as
    pgg_pack_gbuffer from per-pixel kind / albedo / roughness -- misses
    (mat -1) included; the e2e bench leg uploads this form."""
    import torch

    from paper_2112_09728_b200 import synth
    from paper_2112_09728_b200.layout import GBufferPlanes
    (_, _), (g, _) = list(synth.sequence(320, 180, 2, seed=3, device=cuda_dev))
    assert (g["mat"] < 0).any() and (g["has_history"]).any()
    a = GBufferPlanes.from_ref(g, device=cuda_dev)
    kind, rough, alb = synth.materials(3, cuda_dev)
    b = GBufferPlanes.pack_mat(g["valid"], g["pos"], g["normal"], g["depth"], g["mat"], kind, alb, rough, g["view"],
                               g["motion"], g["has_history"], g["cam_origin"], device=cuda_dev)
    for k in ("flags", "nd", "pr", "va", "am"):
        assert torch.equal(getattr(a, k), getattr(b, k)), k
