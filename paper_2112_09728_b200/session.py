"""Device-resident guiding pass: the frame loop of pg/cli.py:114-142
(RenderSession.run_frame) on the GPU.

``run_pass`` issues one fused kernel (libpgg ``pgg_guiding_pass``) over a
row band: reproject Gamma along motion vectors (optional), depth-0
guided/BRDF sampling (optional), one EM epoch over the VPL disk (optional).
``GuidingSession`` owns the double-buffered Gamma planes and the previous
G-buffer so a renderer feeds one frame at a time.
"""

import ctypes
from dataclasses import dataclass
from typing import Optional

import torch

from . import _lib
from .layout import GammaPlanes, GBufferPlanes, PassConfig, SamplePlanes, VplPlanes, make_config


@dataclass
class PassResult:
    gamma: Optional[GammaPlanes] = None          # trained Gamma' (EM output)
    gamma_reproj: Optional[GammaPlanes] = None   # reprojected Gamma (input of sampling/EM)
    samples: Optional[SamplePlanes] = None


def run_pass(cfg: PassConfig, frame: int, cur: GBufferPlanes, gamma_prev: GammaPlanes,
             prev: Optional[GBufferPlanes] = None, vpl: Optional[VplPlanes] = None, *, height=None, row0=0,
             rows=None, want_reproj=False, want_samples=True, out_gamma: Optional[GammaPlanes] = None,
             out_reproj: Optional[GammaPlanes] = None, out_samples: Optional[SamplePlanes] = None,
             halo_misses: Optional[torch.Tensor] = None, stream=None) -> PassResult:
    """One launch of the fused pass over rows [row0, row0 + rows) of a frame
    of ``height`` rows (defaults: the whole of ``cur``)."""
    dev = cur.flags.device
    W = cur.width
    H = int(height if height is not None else (cur.height or cur.row0 + cur.rows))
    rows = int(rows if rows is not None else cur.row0 + cur.rows - row0)
    c = make_config(cfg, W, H, frame, row0=row0, rows=rows,
                    prev_cam=prev.cam_origin if prev is not None else (0.0, 0.0, 0.0))
    res = PassResult()
    if want_reproj:
        res.gamma_reproj = out_reproj if out_reproj is not None else GammaPlanes.empty(rows, W, dev, row0)
    if want_samples:
        res.samples = out_samples if out_samples is not None else SamplePlanes.empty(rows, W, cfg.spp, dev)
    if vpl is not None:
        res.gamma = out_gamma if out_gamma is not None else GammaPlanes.empty(rows, W, dev, row0)
    ref = ctypes.byref
    cur_abi = cur.as_abi()
    prev_abi = prev.as_abi() if prev is not None else None
    gin = gamma_prev.as_in()
    vpl_abi = vpl.as_abi() if vpl is not None else None
    grep = res.gamma_reproj.as_out() if want_reproj else None
    gout = res.gamma.as_out() if vpl is not None else None
    smp = res.samples.as_abi() if want_samples else None
    # launch on the tensors' device (and its current stream by default), not
    # on whatever device the calling thread has current
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().pgg_guiding_pass(
            ref(c), ref(cur_abi), ref(prev_abi) if prev_abi is not None else None, ref(gin),
            ref(vpl_abi) if vpl_abi is not None else None, ref(grep) if grep is not None else None,
            ref(gout) if gout is not None else None, ref(smp) if smp is not None else None,
            _lib.ptr(halo_misses), _lib.stream_ptr(stream, dev)))
    return res


class GuidingSession:
    """Frame-sequential guiding state on one GPU (pg/cli.py:92-142, pg mode).

    ``step(gbuf, vpl, frame)`` runs reproject -> sample -> train for one frame
    with Gamma double-buffered in HBM; the previous G-buffer is kept for the
    next frame's reprojection.  Gamma starts as init_stats (or a checkpoint).
    """

    def __init__(self, width, height, cfg: Optional[PassConfig] = None, device="cuda", gamma=None):
        self.width, self.height = int(width), int(height)
        self.cfg = cfg or PassConfig()
        self.device = torch.device(device)
        if gamma is None:
            self.gamma = GammaPlanes.fresh(self.height, self.width, self.device)
        else:
            self.gamma = gamma
        self._spare = GammaPlanes.empty(self.height, self.width, self.device)
        self.prev = None
        self.samples = SamplePlanes.empty(self.height, self.width, self.cfg.spp, self.device)
        self.halo_misses = torch.zeros(1, dtype=torch.int32, device=self.device)

    def step(self, gbuf: GBufferPlanes, vpl: VplPlanes, frame: int, want_samples=True, stream=None):
        res = run_pass(self.cfg, frame, gbuf, self.gamma, prev=self.prev, vpl=vpl, height=self.height,
                       want_samples=want_samples, out_gamma=self._spare,
                       out_samples=self.samples if want_samples else None, halo_misses=self.halo_misses,
                       stream=stream)
        self._spare, self.gamma = self.gamma, res.gamma
        self.prev = gbuf
        return res
