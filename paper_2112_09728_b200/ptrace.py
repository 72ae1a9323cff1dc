"""Render-side types and the guided first-bounce sampler; drop-in for the
parts of pgtrace.ptrace on the guiding path (pg/ptrace.py:27-73, 161-220).

The ray-traced render pass itself (gbuffer_pass, _trace_lanes, ...) is
outside this framework's scope: a renderer hands over
its G-buffer and VPL buffer in these types, or in the packed device layout
of layout.py.
"""

from dataclasses import dataclass, field
from typing import NamedTuple, Optional

import numpy as np
import torch

from . import _conv, mixture
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
    if st.shape[0] != n:
        raise ValueError("stats must hold one row per lane")
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
