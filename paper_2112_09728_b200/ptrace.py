"""Drop-in for pgtrace.ptrace (pg/ptrace.py): render-side types, the
guided first-bounce sampler (pg/ptrace.py:161-220) and the render pass that
feeds the guiding pass -- gbuffer_pass, motion_vectors and render_frame
(pg/ptrace.py:97-150, 382-586) -- on the GPU kernels of csrc/pgg_render.cu.

These wrappers take and return the reference's NumPy types; the
device-resident path (no host copies) is render.py + cli.RenderSession.
"""

from dataclasses import dataclass, field
from typing import NamedTuple, Optional

import numpy as np
import torch

from . import _conv, mixture
from . import scene as sc
from .layout import GammaPlanes, GBufferPlanes, PassConfig, SamplePlanes
from .session import run_pass

_EZ = np.array([0.0, 0.0, 1.0])


@dataclass
class PathConfig:
    """(pg/ptrace.py:27-39)"""

    max_depth: int = 4
    nee: bool = True
    guiding: bool = False
    roughness_min_guide: float = 0.05
    spp: int = 1

    def __post_init__(self):
        if self.guiding and self.max_depth < 2:
            raise ValueError("guiding needs max_depth >= 2 (the first bounce must exist)")
        if self.spp < 1 or self.max_depth < 1:
            raise ValueError("spp and max_depth must be >= 1")


@dataclass
class GBuffer:
    """Primary-hit record per pixel (pg/ptrace.py:42-64)."""

    width: int
    height: int
    valid: object
    pos: object
    normal: object
    depth: object
    mat: object
    kind: object
    albedo: object
    roughness: object
    front: object
    view: object
    motion: object
    has_history: object
    cam_origin: object


class VplBuffer(NamedTuple):
    """Per-pixel virtual point light (pg/ptrace.py:67-73)."""

    valid: object
    y: object
    radiance: object
    strategy: object


def _sample_first_bounce(scene, idx, pos, nrm, mat, wo, stats, lobe, guided, streams):
    """First scattering direction per lane (pg/ptrace.py:161-220) on the GPU.

    Plain lanes sample the BRDF about the world normal; guided lanes sample
    the mixture in the tangent frame and divide by the full mixture pdf.
    ``streams[idx]`` are advanced in place.  Returns world (wi, pdf, strat, valid).
    """
    torch_in = _conv.is_torch(pos, nrm, wo, stats, streams)
    idx_np = idx.cpu().numpy() if torch.is_tensor(idx) else np.asarray(idx)
    mat_np = mat.cpu().numpy() if torch.is_tensor(mat) else np.asarray(mat)
    kind = np.asarray(scene.mat_kind)[mat_np]
    rough = np.asarray(scene.mat_rough)[mat_np]
    n = len(idx_np)
    st = _conv.to_dev(stats, torch.float64).reshape(-1, 8)
    if st.shape[0] < n:
        raise ValueError("stats must hold at least one row per lane of idx")
    if st.shape[0] > n:
        # pg/ptrace.py:288-290 passes the chunk's per-lane stats / lobe for ALL
        # lanes while idx lists only the active ones, and pg/ptrace.py:205-213
        # indexes them by position within idx (stats[gsel], gsel relative to
        # idx): lane idx[j] uses row j.  With primary-ray misses that pairs a
        # lane with another pixel's mixture; reproduced here so the drop-in
        # returns what the reference returns (the fused pass and the GPU
        # render use every pixel's own Gamma).
        st = st[:n]
        lobe = type(lobe)(*[x[:n] for x in lobe])
    if torch.is_tensor(streams):
        states = streams.view(torch.int64)[torch.as_tensor(idx_np, device=streams.device)].contiguous()
    else:
        states = _conv.u64_to_dev(np.asarray(streams)[idx_np])
    d, t = mixture.sample_lanes(True, nrm, wo, kind, rough, guided, st[:, mixture.MIX_PI], mixture._lobe6(lobe),
                                states)
    if torch.is_tensor(streams):
        streams.view(torch.int64)[torch.as_tensor(idx_np, device=streams.device)] = states
    else:
        np.asarray(streams)[idx_np] = states.cpu().numpy().view(np.uint64)
    wi = d[:, :3].to(torch.float64)
    pdf = d[:, 3].to(torch.float64)
    strat = (t & 1)
    valid = ((t >> 1) & 1).bool()
    if torch_in:
        return wi, pdf, strat, valid
    return wi.cpu().numpy(), pdf.cpu().numpy(), strat.cpu().numpy().astype(np.uint8), valid.cpu().numpy()


def sample_first_bounce_frame(gamma_stats, gbuf, seed, frame_index, spp=1, nee_draws=3, roughness_min_guide=0.05):
    """Depth-0 samples of every valid pixel x spp lane, exactly as the render
    pass issues them (pg/ptrace.py:449-475): lane key pixel*spp+s, ``nee_draws``
    NEE draws first, guided iff valid & (diffuse | rough >= min) & k >= 1.

    Returns dict of (H*W, spp[, 3]) arrays wi, pdf, strategy, valid (NumPy
    unless the stats are a CUDA tensor)."""
    torch_in = _conv.is_torch(gamma_stats)
    dev = _conv.device()
    gb = GBufferPlanes.from_ref(gbuf, device=dev)
    g = GammaPlanes.from_aos(gamma_stats, dev)
    cfg = PassConfig(seed=seed, spp=spp, nee_draws=nee_draws, roughness_min_guide=roughness_min_guide)
    res = run_pass(cfg, frame_index, gb, g, want_samples=True)
    h, w = gb.rows, gb.width
    d = res.samples.dir.reshape(h * w, spp, 4)
    t = res.samples.tag.reshape(h * w, spp)
    out = dict(wi=d[..., :3].to(torch.float64), pdf=d[..., 3].to(torch.float64), strategy=t & 1,
               valid=((t >> 1) & 1).bool())
    if torch_in:
        return out
    return {k: v.cpu().numpy() for k, v in out.items()}


# ---------------------------------------------------------------------------
# render pass (pg/ptrace.py:76-150, 382-586)

@dataclass
class RenderResult:
    """(pg/ptrace.py:76-86)"""

    image: np.ndarray
    vpl: VplBuffer
    gbuffer: GBuffer
    mean_path_length: float
    nonfinite_count: int
    lum_mean: Optional[np.ndarray] = None
    lum_var: Optional[np.ndarray] = None


def _device_scene(scene):
    from .render import device_scene
    return device_scene(scene, _conv.device())


def gbuffer_from_planes(fgb, cam_origin):
    """Packed device G-buffer -> reference GBuffer (float64 NumPy fields).
    Invalid pixels carry the reference's values: pos = origin + inf * dir
    (non-finite), zero normal/depth/material fields, mat -1."""
    g = fgb.planes
    h, w = g.rows, g.width
    fl = g.flags.cpu().numpy()
    nd = g.nd.cpu().numpy().astype(np.float64)
    pr = g.pr.cpu().numpy().astype(np.float64)
    va = g.va.cpu().numpy().astype(np.float64)
    am = g.am.cpu().numpy().astype(np.float64)
    valid = (fl & 1).astype(bool)
    view = va[..., :3]
    pos = pr[..., :3].copy()
    with np.errstate(invalid="ignore", over="ignore"):
        pos[~valid] = np.asarray(cam_origin, dtype=np.float64) + np.inf * (-view[~valid])
    mat = fgb.mat.cpu().numpy().astype(np.int32)
    return GBuffer(
        width=w, height=h, valid=valid, pos=pos, normal=nd[..., :3].copy(), depth=nd[..., 3].copy(), mat=mat,
        kind=((fl >> 2) & 1).astype(np.int32), albedo=np.stack([va[..., 3], am[..., 0], am[..., 1]], axis=-1),
        roughness=pr[..., 3].copy(), front=((fl >> 3) & 1).astype(bool), view=view.copy(),
        motion=np.stack([am[..., 2], am[..., 3]], axis=-1), has_history=((fl >> 1) & 1).astype(bool),
        cam_origin=np.asarray(cam_origin, dtype=np.float64).copy())


def gbuffer_pass(scene, frame_index, resolution):
    """One primary ray through each pixel centre (pg/ptrace.py:97-129), on
    the GPU; float32 fields upcast to float64 NumPy."""
    from .render import gbuffer_planes
    width, height = resolution
    cam = sc.camera_at(scene, frame_index)
    fgb = gbuffer_planes(_device_scene(scene), cam, int(width), int(height))
    return gbuffer_from_planes(fgb, cam.origin)


def motion_vectors(prev_cam, cur_cam, gbuf):
    """Offsets to the previous camera's projection of every valid hit
    (pg/ptrace.py:132-150; pg/scene.py:138-151): one float64 lane kernel
    (pgg_motion_vectors) over the caller's G-buffer."""
    import ctypes

    from . import _lib
    from .render import camera_abi
    h, w = gbuf.height, gbuf.width
    pos = _conv.to_dev(gbuf.pos, torch.float64).reshape(h, w, 3).contiguous()
    valid = _conv.to_dev(gbuf.valid, torch.bool).reshape(h, w).to(torch.uint8).contiguous()
    m = torch.empty(h, w, 2, dtype=torch.float64, device=pos.device)
    has = torch.empty(h, w, dtype=torch.uint8, device=pos.device)
    c = camera_abi(prev_cam)
    _lib.check(_lib.lib().pgg_motion_vectors(ctypes.byref(c), int(w), int(h), _lib.ptr(pos), _lib.ptr(valid),
                                             _lib.ptr(m), _lib.ptr(has), _lib.stream_ptr()))
    has = has.bool()
    if _conv.is_torch(gbuf.pos):
        return m, has
    return m.cpu().numpy(), has.cpu().numpy()


def _planes_from_gbuffer(gbuf, dev):
    """Reference GBuffer -> FrameGBuffer (packed planes + front bit + mat)."""
    from .render import FrameGBuffer
    planes = GBufferPlanes.from_ref(gbuf, device=dev)
    front = _conv.to_dev(gbuf.front, torch.uint8)
    planes.flags |= (front & 1) << 3
    planes.height = int(gbuf.height)
    mat = _conv.to_dev(gbuf.mat, torch.int32)
    return FrameGBuffer(planes, mat)


def render_frame(scene, frame_index, guiding_stats, cfg, seed, resolution=None, gbuf=None, want_moments=False):
    """Render one frame on the GPU (pg/ptrace.py:496-586): pt mode traces
    BRDF lanes; pg mode (cfg.guiding with stats) first runs the guiding
    pass's depth-0 sampler on the Gamma, then traces from its samples."""
    from .render import render_planes
    if gbuf is None:
        if resolution is None:
            raise ValueError("render_frame needs either a G-buffer or a resolution")
        gbuf = gbuffer_pass(scene, frame_index, resolution)
    h, w = gbuf.height, gbuf.width
    guided = bool(cfg.guiding and guiding_stats is not None)
    if guided:
        gs = guiding_stats
        if (gs.numel() if torch.is_tensor(gs) else np.asarray(gs).size) != h * w * 8:
            raise ValueError("guiding buffer dimensions do not match the resolution")
    dev = _conv.device()
    dsc = _device_scene(scene)
    fgb = _planes_from_gbuffer(gbuf, dev)
    depth0 = None
    if guided:
        stats = _conv.to_dev(guiding_stats, torch.float32).reshape(h, w, 8)
        pc = PassConfig(seed=seed, spp=cfg.spp, nee_draws=3 if (cfg.nee and scene.num_emitters) else 0,
                        roughness_min_guide=cfg.roughness_min_guide)
        depth0 = run_pass(pc, frame_index, fgb.planes, GammaPlanes.from_aos(stats, dev), want_samples=True).samples
    rp = render_planes(dsc, fgb, frame_index, seed, spp=cfg.spp, max_depth=cfg.max_depth, nee=cfg.nee,
                       depth0=depth0, want_moments=want_moments)
    return result_from_planes(rp, gbuf, cfg.spp, want_moments)


def result_from_planes(rp, gbuf, spp, want_moments):
    """RenderPlanes -> reference RenderResult (NumPy)."""
    h, w = rp.image.shape[:2]
    cnt = rp.counters.cpu().numpy()
    vy = rp.vpl.y.cpu().numpy().astype(np.float64)
    vl = rp.vpl.L.cpu().numpy()
    code = vl[..., 3].astype(np.int32)
    vpl = VplBuffer(valid=(code & 1).astype(bool), y=vy[..., :3].copy(), radiance=vl[..., :3].astype(np.float64),
                    strategy=(code >> 1).astype(np.uint8))
    out = RenderResult(image=rp.image.cpu().numpy(), vpl=vpl, gbuffer=gbuf,
                       mean_path_length=1.0 + float(cnt[0]) / max(h * w * spp, 1), nonfinite_count=int(cnt[1]))
    if want_moments:
        lm = rp.lum.cpu().numpy()
        n = float(spp)
        out.lum_mean = lm[..., 0] / n
        out.lum_var = np.maximum(lm[..., 1] / n - out.lum_mean ** 2, 0.0) * (n / max(n - 1.0, 1.0))
    return out


# ---------------------------------------------------------------------------
# per-pixel API (pg/ptrace.py:79-95, 336-376)

def worker_count():
    """Host worker threads of the reference's CPU render (PG_THREADS, else
    the CPU count; pg/ptrace.py:89-95).  The GPU render ignores it."""
    import os
    env = os.environ.get("PG_THREADS", "")
    if env.strip():
        try:
            return max(1, int(env))
        except ValueError:
            pass
    return max(1, os.cpu_count() or 1)


class PixelHit(NamedTuple):
    """Single-pixel view of a G-buffer entry (pg/ptrace.py:336-345)."""

    valid: bool
    pos: np.ndarray
    normal: np.ndarray
    mat: int
    roughness: float
    front: bool
    view: np.ndarray


_PCG_MUL, _PCG_INC, _M64 = 6364136223846793005, 1442695040888963407, (1 << 64) - 1


def trace_pixel(scene, gpx, guiding_entry, cfg, streams):
    """One path sample for one pixel (pg/ptrace.py:348-376) through the same
    device kernels as whole frames: the render kernel on a 1x1 G-buffer with
    the caller's PCG32 state (``streams``, one uint64, advanced in place);
    ``guiding_entry`` = (stats (8,), GaussianLobe) samples depth 0 from the
    mixture.  Returns (color (3,), vpl dict); color and VPL come back in the
    float32 device layout."""
    from .render import FrameGBuffer, render_planes
    dev = _conv.device()
    valid = bool(gpx.valid)
    mat = int(gpx.mat) if valid else 0
    kind = int(scene.mat_kind[mat])
    f64 = lambda v: np.asarray(v, dtype=np.float64).reshape(3)  # noqa: E731
    pos, nrm, view = f64(gpx.pos), f64(gpx.normal), f64(gpx.view)
    planes = GBufferPlanes.pack(np.array([[valid]]), pos.reshape(1, 1, 3), nrm.reshape(1, 1, 3), np.zeros((1, 1)),
                                np.array([[kind]]), np.asarray(scene.mat_albedo[mat]).reshape(1, 1, 3),
                                np.array([[float(gpx.roughness)]]), view.reshape(1, 1, 3), device=dev)
    planes.flags |= (1 if (valid and bool(gpx.front)) else 0) << 3
    planes.height = 1
    fgb = FrameGBuffer(planes, torch.tensor([[mat if valid else -1]], dtype=torch.int32, device=dev))
    st0 = int(np.asarray(streams, dtype=np.uint64).reshape(-1)[0]) if not torch.is_tensor(streams) else \
        int(streams.reshape(-1)[0].item()) & _M64
    depth0 = None
    if guiding_entry is not None and valid:
        stats, lobe = guiding_entry
        stats = np.asarray(stats, dtype=np.float64).reshape(8)
        rough_ok = kind == sc.DIFFUSE or float(gpx.roughness) >= cfg.roughness_min_guide
        if rough_ok and stats[mixture.EPOCH] >= 1.0:
            s1 = st0
            for _ in range(3 if (cfg.nee and scene.num_emitters) else 0):
                s1 = (s1 * _PCG_MUL + _PCG_INC) & _M64
            lb = mixture.GaussianLobe(np.asarray(lobe.mu, dtype=np.float64).reshape(1, 2),
                                      np.asarray(lobe.cov, dtype=np.float64).reshape(1, 2, 2),
                                      np.asarray(lobe.chol, dtype=np.float64).reshape(1, 2, 2),
                                      np.atleast_1d(np.asarray(lobe.trunc_z, dtype=np.float64)))
            states1 = torch.tensor([s1 - (1 << 64) if s1 >= (1 << 63) else s1], dtype=torch.int64, device=dev)
            d, t = mixture.sample_lanes(True, nrm.reshape(1, 3), view.reshape(1, 3), np.array([kind]),
                                        np.array([scene.mat_rough[mat]]), np.array([1]), np.array([stats[6]]),
                                        mixture._lobe6(lb), states1)
            depth0 = SamplePlanes(d.reshape(1, 1, 1, 4).contiguous(), t.reshape(1, 1, 1).contiguous(), 1)
    states = torch.tensor([st0 - (1 << 64) if st0 >= (1 << 63) else st0], dtype=torch.int64, device=dev)
    rp = render_planes(_device_scene(scene), fgb, 0, 0, spp=1, max_depth=cfg.max_depth, nee=cfg.nee, depth0=depth0,
                       states=states)
    st_out = int(states[0].item()) & _M64
    if torch.is_tensor(streams):
        streams.reshape(-1)[0] = st_out - (1 << 64) if st_out >= (1 << 63) else st_out
    else:
        np.asarray(streams).reshape(-1)[0] = np.uint64(st_out)
    color = rp.image[0, 0].to(torch.float64).cpu().numpy()
    vy = rp.vpl.y[0, 0].to(torch.float64).cpu().numpy()
    vl = rp.vpl.L[0, 0].to(torch.float64).cpu().numpy()
    code = int(vl[3])
    return color, {"valid": bool(code & 1), "y": vy[:3], "radiance": vl[:3], "strategy": code >> 1}
