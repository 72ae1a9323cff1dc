"""GPU parity of the fused guiding pass (libpgg.so on a B200) against the
reference golden vectors and the CPU oracle.  Tolerances: SURVEY.md 8a."""

import numpy as np
import pytest
import torch

import golden_io as gio
from oracle import pgg_oracle as O
from test_hostcheck import check_gamma, check_samples

pytestmark = pytest.mark.gpu


def _api():
    from paper_2112_09728_b200.layout import GammaPlanes, GBufferPlanes, PassConfig, VplPlanes
    from paper_2112_09728_b200.session import run_pass
    return GammaPlanes, GBufferPlanes, PassConfig, VplPlanes, run_pass


def _samples(res, n, spp):
    d = res.samples.dir.cpu().numpy().reshape(n, spp, 4)
    t = res.samples.tag.cpu().numpy().reshape(n, spp)
    return dict(wi=d[..., :3].astype(np.float64), pdf=d[..., 3].astype(np.float64), strategy=t & 1,
                valid=((t >> 1) & 1).astype(bool))


@pytest.mark.parametrize("f", range(6))
def test_seq_frame(cuda_dev, f):
    GammaPlanes, GBufferPlanes, PassConfig, VplPlanes, run_pass = _api()
    z = gio.load("seq_64x48.npz")
    spp, seed = int(z["spp"]), int(z["seed"])
    cfg = PassConfig(seed=seed, spp=spp)
    cur = GBufferPlanes.from_ref(gio.gbuf_raw(z, f"f{f}_"), device=cuda_dev)
    miss = torch.zeros(1, dtype=torch.int32, device=cuda_dev)
    if f > 0:
        prev = GBufferPlanes.from_ref(gio.gbuf_raw(z, f"f{f-1}_"), device=cuda_dev)
        r = run_pass(cfg, f, cur, GammaPlanes.from_aos(z[f"f{f}_gamma_in"], cuda_dev), prev=prev,
                     want_reproj=True, want_samples=False, halo_misses=miss)
        check_gamma(r.gamma_reproj.to_aos().cpu().numpy(), z[f"f{f}_gamma_reproj"])
    r = run_pass(cfg, f, cur, GammaPlanes.from_aos(z[f"f{f}_gamma_reproj"], cuda_dev),
                 vpl=VplPlanes.from_ref(gio.vpl_raw(z, f"f{f}_"), device=cuda_dev), halo_misses=miss)
    s = _samples(r, 64 * 48, spp)
    check_samples(s, z[f"f{f}_smp_wi"], z[f"f{f}_smp_pdf"], z[f"f{f}_smp_strategy"], z[f"f{f}_smp_valid"])
    check_gamma(r.gamma.to_aos().cpu().numpy(), z[f"f{f}_gamma_trained"])
    assert int(miss.item()) == 0


def test_trained_frame(cuda_dev):
    GammaPlanes, GBufferPlanes, PassConfig, VplPlanes, run_pass = _api()
    z = gio.load("trained_48x40.npz")
    spp, seed, fr = int(z["spp"]), int(z["seed"]), int(z["frame"])
    cur = GBufferPlanes.from_ref(gio.gbuf_raw(z, "c_"), device=cuda_dev)
    prev = GBufferPlanes.from_ref(gio.gbuf_raw(z, "p_"), device=cuda_dev)
    vpl = VplPlanes.from_ref(gio.vpl_raw(z, "c_"), device=cuda_dev)
    gin = GammaPlanes.from_aos(z["gamma_in"], cuda_dev)
    r = run_pass(PassConfig(seed=seed, spp=spp), fr, cur, gin, prev=prev, want_reproj=True, want_samples=False)
    check_gamma(r.gamma_reproj.to_aos().cpu().numpy(), z["gamma_reproj"])
    r = run_pass(PassConfig(seed=seed, spp=spp), fr, cur, gin, vpl=vpl)
    check_samples(_samples(r, 48 * 40, spp), z["smp_wi"], z["smp_pdf"], z["smp_strategy"], z["smp_valid"])
    check_gamma(r.gamma.to_aos().cpu().numpy(), z["gamma_trained"])
    r = run_pass(PassConfig(seed=seed, spp=spp, k_max=32, neighbor_radius=7.3), fr, cur, gin, vpl=vpl,
                 want_samples=False)
    check_gamma(r.gamma.to_aos().cpu().numpy(), z["gamma_trained_r7"])


def _ulp_perturbed_oracle_agreement(frames_ns, w, h, seed, pseed):
    """The reference's own conditioning on this workload (SURVEY 8a basis,
    drift.py): the oracle chain against the same chain with Gamma channels
    0-5 nudged by one float32 ulp (random sign) after frame 0.  Returns the
    final fraction of channels within 1e-4."""
    a = O.fresh_stats(h * w).reshape(h, w, 8).astype(np.float32)
    b = a.copy()
    prev = None
    rng = np.random.default_rng(pseed)
    for f, (g, v) in enumerate(frames_ns):
        _, _, a = O.guiding_frame(a, prev, g, v, seed, f, spp=1)
        _, _, b = O.guiding_frame(b, prev, g, v, seed, f, spp=1)
        if f == 0:
            sgn = rng.choice([-1.0, 1.0], size=b[..., :6].shape).astype(np.float32)
            b[..., :6] = np.nextafter(b[..., :6], b[..., :6] + sgn)
        prev = g
    return float(np.mean(gio.rel_err(b, a) <= 1e-4))


def test_oracle_chain_160x120(cuda_dev):
    """4-frame fused chain on fresh synthetic inputs vs the oracle's chain
    (SURVEY 8a).  Every frame, the oracle is also run one step from the
    GPU's own previous Gamma: that step must meet the single-kernel policy
    (p99.99 <= 1e-4, max <= 1e-3, k exact) -- the kernel's own error.  The
    chain itself must keep k exact on every pixel and max <= 1e-2, and >= 99.9 %
    of channels within 1e-4 -- or, where the reference's own trajectory is
    less stable than that, as close as the reference is to itself after a
    one-ulp perturbation of Gamma (tools/chain_flips.py, profiles/
    r2_chain_flips_160x120.json: at 160x120 / 4 frames the 1-ulp-perturbed
    reference keeps 99.879-99.888 %, the GPU 99.881 %, with zero discrete
    flips -- no reprojection, reset or k decision differs)."""
    from paper_2112_09728_b200 import synth
    from paper_2112_09728_b200.session import GuidingSession
    GammaPlanes, GBufferPlanes, PassConfig, VplPlanes, run_pass = _api()
    w, h, seed = 160, 120, 9
    frames = list(synth.sequence(w, h, 4, seed=seed))
    sess = GuidingSession(w, h, PassConfig(seed=seed, spp=1), device=cuda_dev)
    gam = O.fresh_stats(h * w).reshape(h, w, 8).astype(np.float32)
    prev_ns = None
    frames_ns = []
    for f, (g, v) in enumerate(frames):
        gpu_in = sess.gamma.to_aos().cpu().numpy()
        res = sess.step(GBufferPlanes.from_ref(g, device=cuda_dev), VplPlanes.from_ref(v, device=cuda_dev), f)
        gn, vn = _ns(g), _ns(v)
        frames_ns.append((gn, vn))
        _, smp, gam = O.guiding_frame(gam, prev_ns, gn, vn, seed, f, spp=1)
        _, asmp, astep = O.guiding_frame(gpu_in, prev_ns, gn, vn, seed, f, spp=1)   # re-anchored step
        prev_ns = gn
        got = sess.gamma.to_aos().cpu().numpy()
        check_gamma(got, astep)
        s = _samples(res, w * h, 1)
        check_samples(s, asmp["wi"], asmp["pdf"], asmp["strategy"], asmp["valid"])
        np.testing.assert_array_equal(got[..., 7], gam[..., 7])  # k exact along the chain
    got = sess.gamma.to_aos().cpu().numpy()
    r = gio.rel_err(got, gam)
    frac = float(np.mean(r <= 1e-4))
    assert r.max() <= 1e-2, r.max()
    if frac < 0.999:
        ref = min(_ulp_perturbed_oracle_agreement(frames_ns, w, h, seed, p) for p in (0, 1))
        assert frac >= ref - 2e-4, (frac, ref)


def test_1080p_determinism_and_bands(cuda_dev):
    """Full-size properties: bitwise determinism across runs, and row-band
    launches (with halos) equal the whole-frame launch bitwise."""
    from paper_2112_09728_b200 import synth
    GammaPlanes, GBufferPlanes, PassConfig, VplPlanes, run_pass = _api()
    w, h = 1920, 1080
    (gp, _), (gc, vc) = list(synth.sequence(w, h, 2, seed=2, device=cuda_dev, first_frame=3))
    cfg = PassConfig(seed=2, spp=1)
    cur = GBufferPlanes.from_ref(gc, device=cuda_dev)
    prev = GBufferPlanes.from_ref(gp, device=cuda_dev)
    vpl = VplPlanes.from_ref(vc, device=cuda_dev)
    g = GammaPlanes.fresh(h, w, cuda_dev)
    g.g1[..., 3] = torch.randint(0, 70, (h, w), device=cuda_dev, dtype=torch.float32)
    a = run_pass(cfg, 4, cur, g, prev=prev, vpl=vpl, want_reproj=True)
    b = run_pass(cfg, 4, cur, g, prev=prev, vpl=vpl, want_reproj=True)
    torch.cuda.synchronize()
    assert torch.equal(a.gamma.g0, b.gamma.g0) and torch.equal(a.gamma.g1, b.gamma.g1)
    assert torch.equal(a.samples.dir, b.samples.dir) and torch.equal(a.samples.tag, b.samples.tag)
    # 3 bands; every input carries all rows (halo = whole frame) but each launch writes only its band
    for r0, r1 in ((0, 377), (377, 700), (700, 1080)):
        c = run_pass(cfg, 4, cur, g, prev=prev, vpl=vpl, row0=r0, rows=r1 - r0, height=h, want_reproj=True)
        assert torch.equal(c.gamma.g0, a.gamma.g0[r0:r1]) and torch.equal(c.gamma.g1, a.gamma.g1[r0:r1])
        assert torch.equal(c.samples.dir, a.samples.dir[r0:r1])
        assert torch.equal(c.gamma_reproj.g0, a.gamma_reproj.g0[r0:r1])
    # sanity: most valid pixels train (k grows by one over the reprojected k)
    grew = (a.gamma.g1[..., 3] == a.gamma_reproj.g1[..., 3] + 1).float()
    valid = (cur.flags & 1).float()
    assert (grew * valid).sum().item() > 0.8 * valid.sum().item()


def test_16_frame_trajectory_vs_oracle(cuda_dev):
    """SURVEY 8a N-frame policy over the BASELINE sequence length (16 frames,
    fresh Gamma, panning camera with disocclusions): >= 99.9 % of Gamma
    channels within 1e-4 relative, max <= 1e-2, k exact, strategy tags
    >= 99.99 % (discrete masks of a drifting trajectory), pdf p99.9 <= 1e-3."""
    from types import SimpleNamespace

    from paper_2112_09728_b200 import synth
    from paper_2112_09728_b200.session import GuidingSession
    GammaPlanes, GBufferPlanes, PassConfig, VplPlanes, run_pass = _api()
    w, h, seed, F = 96, 64, 21, 16
    frames = list(synth.sequence(w, h, F, seed=seed))
    sess = GuidingSession(w, h, PassConfig(seed=seed, spp=1), device=cuda_dev)
    gam = O.fresh_stats(h * w).reshape(h, w, 8).astype(np.float32)
    prev_ns = None

    def ns(d):
        return SimpleNamespace(**{k: (v.numpy().astype(np.float64) if torch.is_tensor(v) and v.dtype == torch.float32
                                      else (v.numpy() if torch.is_tensor(v) else v)) for k, v in d.items()})

    tags, pdf_err = [], []
    for f, (g, v) in enumerate(frames):
        res = sess.step(GBufferPlanes.from_ref(g, device=cuda_dev), VplPlanes.from_ref(v, device=cuda_dev), f)
        gn, vn = ns(g), ns(v)
        _, smp, gam = O.guiding_frame(gam, prev_ns, gn, vn, seed, f, spp=1)
        prev_ns = gn
        s = _samples(res, w * h, 1)
        tags.append(np.mean(s["strategy"] == smp["strategy"]))
        both = s["valid"] & smp["valid"]
        pdf_err.append(gio.rel_err(s["pdf"][both], smp["pdf"][both]))
    got = sess.gamma.to_aos().cpu().numpy()
    r = gio.rel_err(got, gam)
    assert np.mean(r <= 1e-4) >= 0.999 and r.max() <= 1e-2, (np.mean(r <= 1e-4), r.max())
    np.testing.assert_array_equal(got[..., 7], gam[..., 7])
    assert min(tags) >= 0.9999
    assert np.percentile(np.concatenate(pdf_err), 99.9) <= 1e-3


def _ns(d):
    from types import SimpleNamespace
    return SimpleNamespace(**{k: (v.cpu().numpy().astype(np.float64) if torch.is_tensor(v) and v.dtype == torch.float32
                                  else (v.cpu().numpy() if torch.is_tensor(v) else v)) for k, v in d.items()})


BANDS_1080P = ((0, 48), (516, 564), (1032, 1080))  # top edge, middle, bottom edge


@pytest.mark.parametrize("F", [5, 13])
def test_1080p_vs_oracle(cuda_dev, F):
    """The benchmarked configuration (BASELINE configs[1]/[2]: 1920x1080,
    1 spp, reproject + depth-0 sampling/pdf (MIS) + EM, disocclusions from
    the panning camera and the hole pattern) against the CPU oracle on three
    full-width row bands -- the top and bottom frame edges and the middle --
    with the whole frame as context (pg/guide_buffers.py:262-283, 78-137;
    pg/ptrace.py:161-220).  Gamma comes from F - 1 GPU frames of the bench
    sequence (trained lobes: correlated, reset, k up to 4) and is fed to both
    sides (F - 1 = 4 and 12 frames: k up to 4 / 12, EM budgets 20 down to
    17).  Single-kernel policy: Gamma p99.99 <= 1e-4, max <=
    1e-3, k exact; samples: tags and validity exact, directions <= 1e-5,
    pdf p99.99 <= 1e-4."""
    from paper_2112_09728_b200 import synth
    from paper_2112_09728_b200.session import GuidingSession
    GammaPlanes, GBufferPlanes, PassConfig, VplPlanes, run_pass = _api()
    w, h, seed = 1920, 1080, 0
    frames = list(synth.sequence(w, h, F, seed=seed, device=cuda_dev))
    cfg = PassConfig(seed=seed, spp=1)
    sess = GuidingSession(w, h, cfg, device=cuda_dev)
    for f in range(F - 1):
        g, v = frames[f]
        sess.step(GBufferPlanes.from_ref(g, device=cuda_dev), VplPlanes.from_ref(v, device=cuda_dev), f)
    gin = sess.gamma.to_aos().cpu().numpy()
    (gp, _), (gc, vc) = frames[F - 2], frames[F - 1]
    cur = GBufferPlanes.from_ref(gc, device=cuda_dev)
    prev = GBufferPlanes.from_ref(gp, device=cuda_dev)
    miss = torch.zeros(1, dtype=torch.int32, device=cuda_dev)
    r = run_pass(cfg, F - 1, cur, GammaPlanes.from_aos(gin, cuda_dev), prev=prev,
                 vpl=VplPlanes.from_ref(vc, device=cuda_dev), want_reproj=True, halo_misses=miss)
    got_rep = r.gamma_reproj.to_aos().cpu().numpy()
    got = r.gamma.to_aos().cpu().numpy()
    smp = _samples(r, w * h, 1)
    gpn, gcn, vcn = _ns(gp), _ns(gc), _ns(vc)
    rep = O.reproject(gin, gpn, gcn)
    check_gamma(got_rep, rep)  # whole frame
    assert int(miss.item()) == 0
    valid = gcn.valid.astype(bool)
    assert valid.mean() < 0.95 and (gin[..., 7] >= 1).mean() > 0.5  # disocclusions present, history trained
    for r0, r1 in BANDS_1080P:
        _, osmp, otr = O.guiding_frame(gin, gpn, gcn, vcn, seed, F - 1, spp=1, rows=(r0, r1))
        check_gamma(got[r0:r1], otr)
        band = slice(r0 * w, r1 * w)
        check_samples({k: v[band] for k, v in smp.items()}, osmp["wi"], osmp["pdf"], osmp["strategy"],
                      osmp["valid"])



BANDS_4K = ((0, 16), (1072, 1088), (2144, 2160))


def test_4k_4spp_vs_oracle(cuda_dev):
    """BASELINE configs[3]'s pass (3840x2160, 4 spp: four depth-0 lanes per
    pixel, each with its own PCG stream, and their MIS pdfs) against the CPU
    oracle on three full-width 16-row bands (top edge, middle, bottom edge)
    with the whole frame as context, after 4 GPU frames of the 4K sequence.
    Same single-kernel policy as test_1080p_vs_oracle."""
    from paper_2112_09728_b200 import synth
    from paper_2112_09728_b200.session import GuidingSession
    GammaPlanes, GBufferPlanes, PassConfig, VplPlanes, run_pass = _api()
    w, h, seed, spp, F = 3840, 2160, 0, 4, 5
    frames = list(synth.sequence(w, h, F, seed=seed, device=cuda_dev))
    cfg = PassConfig(seed=seed, spp=spp)
    sess = GuidingSession(w, h, cfg, device=cuda_dev)
    for f in range(F - 1):
        g, v = frames[f]
        sess.step(GBufferPlanes.from_ref(g, device=cuda_dev), VplPlanes.from_ref(v, device=cuda_dev), f)
    gin = sess.gamma.to_aos().cpu().numpy()
    (gp, _), (gc, vc) = frames[F - 2], frames[F - 1]
    miss = torch.zeros(1, dtype=torch.int32, device=cuda_dev)
    r = run_pass(cfg, F - 1, GBufferPlanes.from_ref(gc, device=cuda_dev), GammaPlanes.from_aos(gin, cuda_dev),
                 prev=GBufferPlanes.from_ref(gp, device=cuda_dev), vpl=VplPlanes.from_ref(vc, device=cuda_dev),
                 halo_misses=miss)
    got = r.gamma.to_aos().cpu().numpy()
    smp = _samples(r, w * h, spp)
    assert int(miss.item()) == 0
    gpn, gcn, vcn = _ns(gp), _ns(gc), _ns(vc)
    assert (gin[..., 7] >= 1).mean() > 0.5
    for r0, r1 in BANDS_4K:
        _, osmp, otr = O.guiding_frame(gin, gpn, gcn, vcn, seed, F - 1, spp=spp, rows=(r0, r1))
        check_gamma(got[r0:r1], otr)
        band = slice(r0 * w, r1 * w)
        sb = {k: v[band] for k, v in smp.items()}
        assert osmp["wi"].shape == sb["wi"].shape
        check_samples(sb, osmp["wi"], osmp["pdf"], osmp["strategy"], osmp["valid"])
        assert sb["strategy"].any() and not sb["strategy"].all()

def test_1080p_whole_frame_vs_oracle(cuda_dev):
    """Every pixel and lane of the benchmarked 1080p frame (bench sequence
    frame 12: Gamma trained over 12 GPU frames, k up to 12, disocclusions)
    against the CPU oracle (row chunks in a fork pool), SURVEY 8a
    single-kernel policy over the whole frame: Gamma p99.99 <= 1e-4, max <=
    1e-3, k exact; strategy and validity exact; directions <= 1e-5; pdf
    p99.99 <= 1e-4, max <= 1e-3.  tools/full_frame_parity.py runs the same
    for frame 4 and a 4K 4 spp frame (profiles/r2_full_frame_parity.json)."""
    from helpers.full_frame import run
    rec = run(1920, 1080, 1, 13, verbose=False)
    summary = {k: v for k, v in rec.items() if not k.startswith("worst")}
    assert rec["k_mismatches"] == 0 and rec["strategy_mismatches"] == 0 and rec["valid_mismatches"] == 0, summary
    assert rec["gamma_rel_p9999"] <= 1e-4 and rec["gamma_rel_max"] <= 1e-3, summary
    assert rec["dir_abs_max"] <= 1e-5, (summary, rec["worst_dirs"][:2])
    assert rec["pdf_rel_p9999"] <= 1e-4 and rec["pdf_rel_max"] <= 1e-3, summary


@pytest.mark.parametrize("spp,k_max,radius", [(2, 32, 7.3), (3, 16, 12.0)])
def test_whole_frame_other_configs(cuda_dev, spp, k_max, radius):
    """Whole-frame parity at non-default pass parameters (640x360 bench
    sequence, frame 8): EM radius 7.3 / 12 (the shared tile's halo at its
    largest), k_max 32 / 16 (budgets reach their minimum of 5 sooner), 2 / 3
    spp (lane keys pix * spp + s) -- same policy as the 1080p test."""
    from helpers.full_frame import run
    rec = run(640, 360, spp, 9, verbose=False, k_max=k_max, radius=radius, chunk=8)
    summary = {k: v for k, v in rec.items() if not k.startswith("worst")}
    assert rec["k_mismatches"] == 0 and rec["strategy_mismatches"] == 0 and rec["valid_mismatches"] == 0, summary
    assert rec["gamma_rel_p9999"] <= 1e-4 and rec["gamma_rel_max"] <= 1e-3, summary
    assert rec["dir_abs_max"] <= 1e-5, (summary, rec["worst_dirs"][:2])
    assert rec["pdf_rel_p9999"] <= 1e-4 and rec["pdf_rel_max"] <= 1e-3, summary


@pytest.mark.parametrize("name", ["glossy-box", "indirect-corridor"])
def test_whole_frame_rendered_scene(cuda_dev, name):
    """Whole-frame parity on RENDERED inputs (640x360): the GPU frame loop
    runs 3 guided frames of a built-in scene, then frame 3's G-buffer, its
    path-traced VPLs and the trained Gamma go to the fused pass and to the
    oracle -- axis-aligned planar normals, glossy and diffuse materials,
    emitters (NEE draws).  Same policy as the synthetic whole-frame tests
    (tools/scene_parity.py runs the three scenes at 1080p,
    profiles/r2_scene_parity_1080p.json)."""
    from helpers.scene_frame import one
    rec = one(name, F=4, w=640, h=360)
    summary = {k: v for k, v in rec.items() if not k.startswith("worst")}
    assert rec["k_mismatches"] == 0 and rec["strategy_mismatches"] == 0 and rec["valid_mismatches"] == 0, summary
    assert rec["gamma_rel_p9999"] <= 1e-4 and rec["gamma_rel_max"] <= 1e-3, summary
    assert rec["dir_abs_max"] <= 1e-5, summary
    assert rec["pdf_rel_p9999"] <= 1e-4 and rec["pdf_rel_max"] <= 1e-3, summary
