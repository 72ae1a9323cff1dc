"""Edge cases of the fused pass against the oracle: partial
tiles and tiny frames, a neighbour radius beyond the shared-memory tile
(global VPL path), radius 0 (every candidate is the pixel itself), 4 spp,
all-invalid G-buffers, no history, sequences trained past k_max, and VPLs
behind the receiver, in its tangent plane or on it."""

from types import SimpleNamespace

import numpy as np
import pytest
import torch

import golden_io as gio
from oracle import pgg_oracle as O
from test_hostcheck import check_gamma, check_samples

pytestmark = pytest.mark.gpu


def _ns(d):
    return SimpleNamespace(**{k: (v.cpu().numpy().astype(np.float64) if torch.is_tensor(v) and v.dtype == torch.float32
                                  else (v.cpu().numpy() if torch.is_tensor(v) else v)) for k, v in d.items()})


def _inputs(w, h, seed, first=3):
    from paper_2112_09728_b200 import synth
    (gp, _), (gc, vc) = list(synth.sequence(w, h, 2, seed=seed, first_frame=first))
    rng = np.random.default_rng(seed)
    st = O.fresh_stats(h * w).reshape(h, w, 8)
    st[..., 0:2] = rng.uniform(0.2, 0.8, (h, w, 2))
    sd = rng.uniform(0.03, 0.3, (h, w, 2))
    rho = rng.uniform(-0.8, 0.8, (h, w))
    st[..., 2] = sd[..., 0] ** 2 + st[..., 0] ** 2
    st[..., 3] = sd[..., 1] ** 2 + st[..., 1] ** 2
    st[..., 4] = rho * sd[..., 0] * sd[..., 1] + st[..., 0] * st[..., 1]
    st[..., 6] = rng.uniform(0.05, 0.95, (h, w))
    st[..., 7] = rng.integers(0, 80, (h, w))
    return gp, gc, vc, st.astype(np.float32)


def _run(cuda_dev, gp, gc, vc, st, frame, seed, spp=1, **kw):
    from paper_2112_09728_b200.layout import GammaPlanes, GBufferPlanes, PassConfig, VplPlanes
    from paper_2112_09728_b200.session import run_pass
    cfg = PassConfig(seed=seed, spp=spp, **kw)
    cur = GBufferPlanes.from_ref(gc, device=cuda_dev)
    prev = GBufferPlanes.from_ref(gp, device=cuda_dev) if gp is not None else None
    r = run_pass(cfg, frame, cur, GammaPlanes.from_aos(st, cuda_dev), prev=prev,
                 vpl=VplPlanes.from_ref(vc, device=cuda_dev), want_reproj=True)
    d = r.samples.dir.cpu().numpy().reshape(-1, spp, 4)
    t = r.samples.tag.cpu().numpy().reshape(-1, spp)
    smp = dict(wi=d[..., :3].astype(np.float64), pdf=d[..., 3].astype(np.float64), strategy=t & 1,
               valid=((t >> 1) & 1).astype(bool))
    return r.gamma_reproj.to_aos().cpu().numpy(), smp, r.gamma.to_aos().cpu().numpy()


def _oracle(gp, gc, vc, st, frame, seed, spp=1, **kw):
    return O.guiding_frame(st, _ns(gp) if gp is not None else None, _ns(gc), _ns(vc), seed, frame, spp=spp, **kw)


@pytest.mark.parametrize("w,h", [(33, 9), (1, 1), (31, 1), (70, 17)])
def test_partial_tiles_and_tiny_frames(cuda_dev, w, h):
    gp, gc, vc, st = _inputs(w, h, seed=w * 7 + h)
    got = _run(cuda_dev, gp, gc, vc, st, 4, 5, spp=2)
    ref = _oracle(gp, gc, vc, st, 4, 5, spp=2)
    check_gamma(got[0], ref[0])
    check_samples(got[1], ref[1]["wi"], ref[1]["pdf"], ref[1]["strategy"], ref[1]["valid"])
    check_gamma(got[2], ref[2])


@pytest.mark.parametrize("radius", [15.0, 0.0, 2.5])
def test_radius_paths(cuda_dev, radius):
    """radius > 12 reads VPLs from global memory instead of the TMA tile."""
    gp, gc, vc, st = _inputs(64, 40, seed=3)
    got = _run(cuda_dev, gp, gc, vc, st, 2, 8, neighbor_radius=radius)
    ref = _oracle(gp, gc, vc, st, 2, 8, radius=radius)
    check_gamma(got[2], ref[2])


def test_four_spp(cuda_dev):
    gp, gc, vc, st = _inputs(48, 32, seed=11)
    got = _run(cuda_dev, gp, gc, vc, st, 6, 2, spp=4)
    ref = _oracle(gp, gc, vc, st, 6, 2, spp=4)
    check_samples(got[1], ref[1]["wi"], ref[1]["pdf"], ref[1]["strategy"], ref[1]["valid"])
    check_gamma(got[2], ref[2])


def test_all_invalid_gbuffer(cuda_dev):
    gp, gc, vc, st = _inputs(40, 24, seed=4)
    gc = dict(gc)
    gc["valid"] = torch.zeros_like(gc["valid"])
    got = _run(cuda_dev, gp, gc, vc, st, 3, 1)
    # nothing reprojects, nothing trains: Gamma passes through, samples are zero
    np.testing.assert_array_equal(got[2], got[0])
    assert (got[1]["pdf"] == 0).all() and not got[1]["valid"].any()
    ref = _oracle(gp, gc, vc, st, 3, 1)
    check_gamma(got[0], ref[0])


def test_no_history_resets(cuda_dev):
    gp, gc, vc, st = _inputs(40, 24, seed=6)
    gc = dict(gc)
    gc["has_history"] = torch.zeros_like(gc["has_history"])
    got = _run(cuda_dev, gp, gc, vc, st, 3, 1)
    ref = _oracle(gp, gc, vc, st, 3, 1)
    check_gamma(got[0], ref[0])
    v = gc["valid"].cpu().numpy().astype(bool)
    fresh = O.fresh_stats(1).astype(np.float32)[0]
    assert (got[0][v] == fresh).all()  # every valid pixel starts from init_stats
    check_gamma(got[2], ref[2])


def test_vpls_behind_and_in_the_tangent_plane(cuda_dev):
    """Records the reference masks or re-decides: VPLs straight behind the
    receiver (own record along -n: the square map's 1 + z reaches 0, masked)
    and VPLs in the receiver's tangent plane (cosine ~0: the float64 cosine
    path), mixed with ordinary ones."""
    gp, gc, vc, st = _inputs(48, 32, seed=21)
    vc = dict(vc)
    pos, n = gc["pos"], gc["normal"]
    y = vc["y"].clone()
    h, w = pos.shape[:2]
    sel = torch.zeros(h, w, dtype=torch.long)
    sel[::2, ::2] = 1  # behind
    sel[1::2, 1::2] = 2  # tangent plane: pos + (n x helper) * 1.5
    behind = pos - 2.0 * n
    helper = torch.tensor([0.0, 0.0, 1.0]).expand_as(n)
    t = torch.cross(n, helper, dim=-1)
    t = t / torch.clamp(torch.sqrt((t * t).sum(-1, keepdim=True)), min=1e-12)
    tangent = pos + 1.5 * t
    y = torch.where((sel == 1)[..., None], behind, y)
    y = torch.where((sel == 2)[..., None], tangent, y)
    vc["y"] = y
    got = _run(cuda_dev, gp, gc, vc, st, 4, 9)
    assert np.isfinite(got[2]).all()
    ref = _oracle(gp, gc, vc, st, 4, 9)
    check_gamma(got[2], ref[2])


def test_kmax_saturation(cuda_dev):
    """k beyond k_max: eta = 1/k_max, N = 5 candidates."""
    gp, gc, vc, st = _inputs(48, 32, seed=12)
    st[..., 7] = 500
    got = _run(cuda_dev, gp, gc, vc, st, 5, 3, k_max=16)
    ref = _oracle(gp, gc, vc, st, 5, 3, kmax=16)
    check_gamma(got[2], ref[2])


@pytest.mark.parametrize("gpu_kw,oracle_kw,spp", [
    ({}, {}, 8),                                                            # many lanes per pixel
    ({"nee_draws": 0}, {"nee_draws": 0}, 2),                                # scenes without emitters
    ({"nee_draws": 5}, {"nee_draws": 5}, 1),                                # non-default NEE skip (no jump table)
    ({"k_max": 1}, {"kmax": 1}, 1),                                         # eta = 1, budget 5 from k = 1 on
    ({"depth_rel_tol": 0.01, "normal_dot_min": 0.99},
     {"depth_rel_tol": 0.01, "normal_dot_min": 0.99}, 1),                   # strict reprojection gates
    ({"roughness_min_guide": 0.0}, {"rough_min": 0.0}, 1),                  # every glossy lane guided
    ({"roughness_min_guide": 0.9}, {"rough_min": 0.9}, 1),                  # almost none
    ({"rotate_mean": False}, {"rotate_mean": False}, 1),                    # means carried unrotated
])
def test_pass_parameters_vs_oracle(cuda_dev, gpu_kw, oracle_kw, spp):
    """Non-default pass parameters (pg/cli.py:34-77 RunConfig knobs) through
    the fused pass against the oracle on a 48x40 frame with history: the
    single-kernel policy on the reprojected and trained Gamma and the samples."""
    gp, gc, vc, st = _inputs(48, 40, 7)
    rep, smp, tr = _run(cuda_dev, gp, gc, vc, st, 4, 7, spp=spp, **gpu_kw)
    orep, osmp, otr = _oracle(gp, gc, vc, st, 4, 7, spp=spp, **oracle_kw)
    check_gamma(rep, orep)
    check_gamma(tr, otr)
    check_samples(smp, osmp["wi"].reshape(-1, spp, 3), osmp["pdf"].reshape(-1, spp), osmp["strategy"].reshape(-1, spp),
                  osmp["valid"].reshape(-1, spp))
