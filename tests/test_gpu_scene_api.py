"""GPU batch forms of the scene routines (pg/scene.py:125-414) and the
per-pixel trace (pg/ptrace.py:348-376) against the render oracle / the
whole-frame render: same float64 device code, so results agree to the last
bit except where the oracle's NumPy BLAS dot or libm rounds differently."""

import numpy as np
import pytest

from oracle import pgg_oracle as O
from oracle import pgg_render_oracle as RO

pytestmark = pytest.mark.gpu


def _scene(name="cornell-occluder"):
    from paper_2112_09728_b200 import scene as S
    return S.load_scene(name)


def _rays(n, seed):
    r = np.random.default_rng(seed)
    o = r.uniform(0.05, 1.95, (n, 3))
    d = r.standard_normal((n, 3))
    d /= np.linalg.norm(d, axis=-1, keepdims=True)
    return o, d


def _close(a, b, tol=1e-12):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    fin = np.isfinite(b)
    assert np.array_equal(np.isfinite(a), fin)
    return np.abs(a[fin] - b[fin]) <= tol * np.maximum(1.0, np.abs(b[fin]))


@pytest.mark.parametrize("name", ["cornell-occluder", "glossy-box"])
def test_intersect_and_occluded(cuda_dev, name):
    from paper_2112_09728_b200 import scene as S
    sc = _scene(name)
    o, d = _rays(20000, 1)
    got = S.intersect(sc, o, d)
    ref = RO.cast(sc, o, d)
    agree = got["hit"] == ref.hit
    assert agree.mean() >= 0.9999
    both = got["hit"] & ref.hit
    assert (got["mat"][both] == ref.mat[both]).mean() >= 0.9999
    assert _close(got["t"][both], ref.t[both]).mean() >= 0.999
    assert np.array_equal(got["front"][both], ref.front[both])
    tmax = np.random.default_rng(2).uniform(0.1, 3.0, len(o))
    assert (S.occluded(sc, o, d, tmax) == RO.blocked(sc, o, d, tmax)).mean() >= 0.9999


def test_sample_emitter(cuda_dev):
    from paper_2112_09728_b200 import scene as S
    sc = _scene()
    p = np.random.default_rng(3).uniform(0.1, 1.9, (5000, 3))
    st = O.seed_lanes(9, 2, np.arange(5000), 0)
    st_ref = st.copy()
    w, dist, le, pdf = S.sample_emitter(sc, p, st)
    rw, rdist, rle, rpdf = RO.light_sample(sc, p, st_ref)
    np.testing.assert_array_equal(st, st_ref)
    assert _close(w, rw).all() and _close(dist, rdist).all() and _close(pdf, rpdf).all()
    np.testing.assert_array_equal(le, rle)


def test_brdf_lanes(cuda_dev):
    from paper_2112_09728_b200 import scene as S
    r = np.random.default_rng(4)
    n = 20000
    kind = r.integers(0, 2, n)
    alb = r.uniform(0, 1, (n, 3))
    rough = r.uniform(0.05, 1.0, n)
    nrm = r.standard_normal((n, 3))
    nrm /= np.linalg.norm(nrm, axis=-1, keepdims=True)
    wo = r.standard_normal((n, 3))
    wo /= np.linalg.norm(wo, axis=-1, keepdims=True)
    wo = np.where((np.sum(wo * nrm, -1) < 0)[:, None], -wo, wo)
    wi = r.standard_normal((n, 3))
    wi /= np.linalg.norm(wi, axis=-1, keepdims=True)
    f = S.brdf_eval(kind, alb, rough, wi, wo, nrm)
    assert _close(f, O.brdf_value(kind, alb, rough, wi, wo, nrm), 1e-13).mean() >= 0.9999
    assert _close(S.brdf_pdf(kind, rough, wi, wo, nrm), O.brdf_density(kind, rough, wi, wo, nrm), 1e-13).mean() >= 0.9999
    st = O.seed_lanes(5, 1, np.arange(n), 0)
    st_ref = st.copy()
    w, pdf, ok = S.brdf_sample(kind, alb, rough, wo, nrm, st)
    rw, rpdf, rok = O.brdf_draw(kind, rough, wo, nrm, st_ref)
    np.testing.assert_array_equal(st, st_ref)
    assert (ok == rok).mean() >= 0.9999
    assert _close(w, rw, 1e-12).mean() >= 0.9999
    # GGX pdf near the specular peak amplifies the 1-ulp sin/cos differences of the VNDF draw
    assert _close(pdf[ok & rok], rpdf[ok & rok], 1e-9).mean() >= 0.9999


def test_camera_lanes(cuda_dev):
    from paper_2112_09728_b200 import scene as S
    sc = S.scene_from_dict(S.BUILTIN_SCENES["glossy-box"]())
    cam = S.camera_at(sc, 0)
    py, px = np.meshgrid(np.arange(36, dtype=np.float64), np.arange(52, dtype=np.float64), indexing="ij")
    d = S.primary_ray_dirs(cam, 52, 36, px, py)
    assert _close(d, RO.eye_rays(cam, 52, 36, px, py), 1e-15).all()
    pts = np.random.default_rng(6).uniform(-1, 3, (4000, 3))
    a = S.project_to_pixels(cam, 52, 36, pts)
    b = RO.to_pixels(cam, 52, 36, pts)
    assert np.array_equal(a[2], b[2])
    assert _close(a[0], b[0], 1e-12).all() and _close(a[1], b[1], 1e-12).all()


def test_trace_pixel_matches_frame_lane(cuda_dev):
    """trace_pixel with the frame's own lane stream reproduces that lane of
    render_frame bit for bit (pt), and to sampler precision (pg)."""
    from paper_2112_09728_b200 import mixture, ptrace
    sc = _scene("glossy-box")
    w, h, fr, seed = 24, 18, 2, 3
    gb = ptrace.gbuffer_pass(sc, fr, (w, h))
    rng = np.random.default_rng(7)
    stats = np.zeros((h, w, 8), np.float32)
    stats[..., 0:2] = rng.uniform(0.3, 0.7, (h, w, 2))
    stats[..., 2:4] = stats[..., 0:2] ** 2 + 0.02
    stats[..., 4] = stats[..., 0] * stats[..., 1]
    stats[..., 6] = 0.6
    stats[..., 7] = 3
    for guided in (False, True):
        cfg = ptrace.PathConfig(spp=1, guiding=guided)
        full = ptrace.render_frame(sc, fr, stats if guided else None, cfg, seed, gbuf=gb)
        lb = mixture.lobe_from_stats(stats.reshape(-1, 8).astype(np.float64))
        for (y, x) in [(5, 7), (12, 20), (9, 3), (0, 0)]:
            pix = y * w + x
            st = O.seed_lanes(seed, fr, np.array([pix]), 0)
            gpx = ptrace.PixelHit(bool(gb.valid[y, x]), gb.pos[y, x], gb.normal[y, x], int(gb.mat[y, x]),
                                  float(gb.roughness[y, x]), bool(gb.front[y, x]), gb.view[y, x])
            entry = None
            if guided:
                entry = (stats[y, x], mixture.GaussianLobe(lb.mu[pix], lb.cov[pix], lb.chol[pix], lb.trunc_z[pix]))
            color, vpl = ptrace.trace_pixel(sc, gpx, entry, cfg, st)
            ref = full.image[y, x].astype(np.float64)
            if guided:
                np.testing.assert_allclose(color, ref, rtol=1e-4, atol=1e-6)
            else:
                np.testing.assert_array_equal(color.astype(np.float32), full.image[y, x])
            assert vpl["valid"] == bool(full.vpl.valid[y, x])


def test_device_table_follows_scene_edits(cuda_dev):
    """The cached device copy of a scene is rebuilt when the scene changes."""
    from paper_2112_09728_b200 import scene as S
    sc = _scene()
    o, d = _rays(4000, 9)
    a = S.intersect(sc, o, d)
    sc.sph_radius = sc.sph_radius * 1.5
    b = S.intersect(sc, o, d)
    ref = RO.cast(sc, o, d)
    assert (b["hit"] == ref.hit).mean() >= 0.9999 and (b["mat"] == ref.mat).mean() >= 0.9999
    assert not np.array_equal(a["t"], b["t"])
