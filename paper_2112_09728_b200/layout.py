"""Device-resident buffers of the guiding pass in the packed B200 layout.

Gamma is two float4 planes (g0 = mu_x, mu_y, m2_xx, m2_yy; g1 = m2_xy, w_sum,
pi, k), the G-buffer four float4 planes + a flag byte, Pi two float4 planes
(see include/pgg.h).  Every plane is a contiguous row-major (rows, W[, 4])
torch tensor so 32 consecutive pixels of a warp read 512 contiguous bytes.
Conversion from the reference's AoS / float64 structures happens here, at
the API edge, on the device (pgg_pack_* kernels).
"""

from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _lib

F32 = torch.float32


@dataclass
class GammaPlanes:
    """Gamma of rows [row0, row0 + rows) of a W-wide frame."""

    g0: torch.Tensor  # (rows, W, 4) float32
    g1: torch.Tensor
    row0: int = 0

    @property
    def rows(self):
        return self.g0.shape[0]

    @property
    def width(self):
        return self.g0.shape[1]

    @classmethod
    def empty(cls, rows, width, device, row0=0):
        return cls(torch.empty(rows, width, 4, dtype=F32, device=device),
                   torch.empty(rows, width, 4, dtype=F32, device=device), row0)

    @classmethod
    def fresh(cls, rows, width, device, row0=0, stream=None):
        g = cls.empty(rows, width, device, row0)
        _lib.check(_lib.lib().pgg_gamma_init(rows * width, _lib.ptr(g.g0), _lib.ptr(g.g1), _lib.stream_ptr(stream)))
        return g

    @classmethod
    def from_aos(cls, stats, device="cuda", row0=0, stream=None):
        """(rows, W, 8) float32 array/tensor -> planes."""
        t = torch.as_tensor(np.ascontiguousarray(stats, dtype=np.float32) if isinstance(stats, np.ndarray)
                            else stats).to(device=device, dtype=F32).contiguous()
        rows, w = t.shape[0], t.shape[1]
        g = cls.empty(rows, w, device, row0)
        _lib.check(_lib.lib().pgg_gamma_split(rows * w, _lib.ptr(t), _lib.ptr(g.g0), _lib.ptr(g.g1),
                                              _lib.stream_ptr(stream)))
        return g

    def to_aos(self, stream=None):
        """planes -> (rows, W, 8) float32 tensor on the device."""
        out = torch.empty(self.rows, self.width, 8, dtype=F32, device=self.g0.device)
        _lib.check(_lib.lib().pgg_gamma_join(self.rows * self.width, _lib.ptr(self.g0), _lib.ptr(self.g1),
                                             _lib.ptr(out), _lib.stream_ptr(stream)))
        return out

    def as_in(self):
        return _lib.GammaIn(_lib.ptr(self.g0), _lib.ptr(self.g1), self.row0, self.rows)

    def as_out(self):
        return _lib.GammaOut(_lib.ptr(self.g0), _lib.ptr(self.g1))


@dataclass
class GBufferPlanes:
    """Packed G-buffer rows [row0, row0 + rows) plus the camera origin."""

    flags: torch.Tensor  # (rows, W) uint8
    nd: torch.Tensor     # (rows, W, 4) normal.xyz, depth
    pr: torch.Tensor     # (rows, W, 4) pos.xyz, roughness
    va: torch.Tensor     # (rows, W, 4) view.xyz, albedo.r
    am: torch.Tensor     # (rows, W, 4) albedo.g, albedo.b, motion.xy
    cam_origin: tuple = (0.0, 0.0, 0.0)
    row0: int = 0
    height: Optional[int] = None  # full frame height (defaults to rows)

    @property
    def rows(self):
        return self.flags.shape[0]

    @property
    def width(self):
        return self.flags.shape[1]

    @classmethod
    def empty(cls, rows, width, device, row0=0):
        e = lambda: torch.empty(rows, width, 4, dtype=F32, device=device)  # noqa: E731
        return cls(torch.empty(rows, width, dtype=torch.uint8, device=device), e(), e(), e(), e(), row0=row0)

    @classmethod
    def pack(cls, valid, pos, normal, depth, kind, albedo, roughness, view, motion=None, has_history=None,
             cam_origin=(0.0, 0.0, 0.0), device="cuda", row0=0, stream=None):
        """Reference GBuffer fields (pg/ptrace.py:42-64; NumPy or torch, any
        float dtype) -> packed planes, converted on the device."""
        def dev(a, dt):
            if isinstance(a, np.ndarray):
                a = torch.from_numpy(np.ascontiguousarray(a))
            return a.to(device=device, dtype=dt).contiguous()

        v = dev(valid, torch.uint8)
        rows, w = v.shape
        g = cls.empty(rows, w, device, row0)
        g.cam_origin = tuple(float(c) for c in np.asarray(cam_origin, dtype=np.float64).reshape(3))
        args = [dev(pos, F32), dev(normal, F32), dev(depth, F32), dev(kind, torch.int32), dev(albedo, F32),
                dev(roughness, F32), dev(view, F32),
                dev(motion, F32) if motion is not None else None,
                dev(has_history, torch.uint8) if has_history is not None else None]
        _lib.check(_lib.lib().pgg_pack_gbuffer(rows * w, _lib.ptr(v), *[_lib.ptr(a) for a in args],
                                               _lib.ptr(g.flags), _lib.ptr(g.nd), _lib.ptr(g.pr), _lib.ptr(g.va),
                                               _lib.ptr(g.am), _lib.stream_ptr(stream)))
        return g

    @classmethod
    def pack_mat(cls, valid, pos, normal, depth, mat, mat_kind, mat_albedo, mat_rough, view, motion=None,
                 has_history=None, cam_origin=(0.0, 0.0, 0.0), device="cuda", row0=0, stream=None):
        """Like pack(), from the G-buffer's material ids (-1 = miss) and the
        scene's material table (kind, albedo rgb, roughness per material):
        the lookups of pg/ptrace.py:97-129 done on the device."""
        def dev(a, dt):
            if isinstance(a, np.ndarray):
                a = torch.from_numpy(np.ascontiguousarray(a))
            return a.to(device=device, dtype=dt).contiguous()

        v = dev(valid, torch.uint8)
        rows, w = v.shape
        g = cls.empty(rows, w, device, row0)
        g.cam_origin = tuple(float(c) for c in np.asarray(cam_origin, dtype=np.float64).reshape(3))
        mk, ma, mr = dev(mat_kind, torch.int32), dev(mat_albedo, F32), dev(mat_rough, F32)
        args = [dev(pos, F32), dev(normal, F32), dev(depth, F32), dev(mat, torch.int32)]
        tail = [dev(view, F32), dev(motion, F32) if motion is not None else None,
                dev(has_history, torch.uint8) if has_history is not None else None]
        _lib.check(_lib.lib().pgg_pack_gbuffer_mat(
            rows * w, _lib.ptr(v), *[_lib.ptr(a) for a in args], int(mk.numel()), _lib.ptr(mk), _lib.ptr(ma),
            _lib.ptr(mr), *[_lib.ptr(a) for a in tail], _lib.ptr(g.flags), _lib.ptr(g.nd), _lib.ptr(g.pr),
            _lib.ptr(g.va), _lib.ptr(g.am), _lib.stream_ptr(stream)))
        return g

    @classmethod
    def from_ref(cls, gb, device="cuda", row0=0, stream=None):
        """From a reference-style GBuffer object or dict."""
        get = (lambda k: gb[k]) if isinstance(gb, dict) else (lambda k: getattr(gb, k))
        return cls.pack(get("valid"), get("pos"), get("normal"), get("depth"), get("kind"), get("albedo"),
                        get("roughness"), get("view"), get("motion"), get("has_history"), get("cam_origin"),
                        device=device, row0=row0, stream=stream)

    def as_abi(self):
        return _lib.GBuffer(_lib.ptr(self.flags), _lib.ptr(self.nd), _lib.ptr(self.pr), _lib.ptr(self.va),
                            _lib.ptr(self.am), self.row0, self.rows)


@dataclass
class VplPlanes:
    """Pi rows [row0, row0 + rows): y float4 (pos, usable), L float4 (rgb, 0)."""

    y: torch.Tensor
    L: torch.Tensor
    row0: int = 0

    @property
    def rows(self):
        return self.y.shape[0]

    @classmethod
    def pack(cls, valid, y, radiance, strategy, device="cuda", row0=0, stream=None):
        """VplBuffer fields (pg/ptrace.py:67-73) -> planes."""
        def dev(a, dt):
            if isinstance(a, np.ndarray):
                a = torch.from_numpy(np.ascontiguousarray(a))
            return a.to(device=device, dtype=dt).contiguous()

        v = dev(valid, torch.uint8)
        rows, w = v.shape
        out = cls(torch.empty(rows, w, 4, dtype=F32, device=device), torch.empty(rows, w, 4, dtype=F32, device=device),
                  row0)
        # keep the converted inputs referenced until the launch is enqueued
        # (a freed temporary's block could be handed to the next conversion)
        yy, rr, ss = dev(y, F32), dev(radiance, F32), dev(strategy, torch.uint8)
        _lib.check(_lib.lib().pgg_pack_vpl(rows * w, _lib.ptr(v), _lib.ptr(yy), _lib.ptr(rr), _lib.ptr(ss),
                                           _lib.ptr(out.y), _lib.ptr(out.L), _lib.stream_ptr(stream)))
        return out

    @classmethod
    def from_ref(cls, vpl, device="cuda", row0=0, stream=None):
        get = (lambda k: vpl[k]) if isinstance(vpl, dict) else (lambda k: getattr(vpl, k))
        return cls.pack(get("valid"), get("y"), get("radiance"), get("strategy"), device=device, row0=row0,
                        stream=stream)

    def as_abi(self):
        return _lib.Vpl(_lib.ptr(self.y), _lib.ptr(self.L), self.row0, self.rows)


@dataclass
class SamplePlanes:
    """Depth-0 samples of rows [row0, row0 + rows), lane = pixel * spp + s."""

    dir: torch.Tensor   # (rows, W, spp, 4) wi.xyz, pdf
    tag: torch.Tensor   # (rows, W, spp) uint8: bit0 GAUSSIAN, bit1 valid
    spp: int = 1

    @classmethod
    def empty(cls, rows, width, spp, device):
        return cls(torch.empty(rows, width, spp, 4, dtype=F32, device=device),
                   torch.empty(rows, width, spp, dtype=torch.uint8, device=device), spp)

    def as_abi(self):
        return _lib.Samples(_lib.ptr(self.dir), _lib.ptr(self.tag))

    @property
    def wi(self):
        return self.dir[..., :3]

    @property
    def pdf(self):
        return self.dir[..., 3]

    @property
    def strategy(self):
        return self.tag & 1

    @property
    def valid(self):
        return (self.tag >> 1) & 1


@dataclass
class PassConfig:
    """Knobs of the pass (defaults = the reference's, pg/cli.py:34-77)."""

    seed: int = 0
    spp: int = 1
    nee_draws: int = 3
    k_max: int = 64
    neighbor_radius: float = 10.0
    depth_rel_tol: float = 0.1
    normal_dot_min: float = 0.9
    rotate_mean: bool = True
    roughness_min_guide: float = 0.05
    extra: dict = field(default_factory=dict)


def make_config(cfg: PassConfig, width, height, frame, row0=0, rows=None, prev_cam=(0.0, 0.0, 0.0)):
    c = _lib.Config()
    c.width, c.height = int(width), int(height)
    c.row0 = int(row0)
    c.rows = int(height - row0 if rows is None else rows)
    c.spp = int(cfg.spp)
    c.nee_draws = int(cfg.nee_draws)
    c.k_max = int(cfg.k_max)
    c.rotate_mean = 1 if cfg.rotate_mean else 0
    c.radius = float(cfg.neighbor_radius)
    c.depth_rel_tol = float(cfg.depth_rel_tol)
    c.normal_dot_min = float(cfg.normal_dot_min)
    c.rough_min_guide = float(cfg.roughness_min_guide)
    for i in range(3):
        c.prev_cam[i] = float(prev_cam[i])
    c.key_sample = _lib.frame_key(cfg.seed, frame, 0)
    c.key_train = _lib.frame_key(cfg.seed, frame, 1)
    return c
