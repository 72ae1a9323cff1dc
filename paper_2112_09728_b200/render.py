"""Device-resident render pass: the producer of the guiding pass's inputs
(SURVEY.md 8f rank 1).  Two kernels of libpgg (csrc/pgg_render.cu):

* ``gbuffer_planes`` — primary ray per pixel centre into the packed G-buffer
  planes + material ids, with the camera motion vectors of the previous
  frame fused in (pg/ptrace.py:97-150).
* ``render_planes`` — spp path lanes per pixel with NEE at every vertex,
  writing the image, the VPL planes the EM pass reads, luminance moments
  and path counters (pg/ptrace.py:223-355, 382-586).  In pg mode the depth-0
  scatter is the guiding pass's sample (``SamplePlanes`` of
  ``session.run_pass``), exactly the division of work of pg/ptrace.py:288.

Everything stays in HBM; NumPy conversion happens only in the
reference-shaped wrappers of ptrace.py.
"""

import ctypes
from dataclasses import dataclass
from typing import Optional

import torch

from . import _lib
from .layout import GBufferPlanes, SamplePlanes, VplPlanes


class DeviceScene:
    """A Scene's packed float64 table resident on the device (pgg_scene)."""

    def __init__(self, scene, device=None, packed=None):
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        table, (nm, ns, nq, ne) = packed if packed is not None else scene.pack()
        self.key = table.tobytes()
        self.scene = scene
        self.table = torch.from_numpy(table).to(dev)
        self.abi = _lib.Scene(_lib.ptr(self.table), nm, ns, nq, ne)
        for i in range(3):
            self.abi.background[i] = float(scene.background[i])
        self.num_emitters = ne
        self.device = dev


def device_scene(scene, device):
    """The scene's device table, cached on the Scene object and rebuilt when
    the scene's contents (or the device) change."""
    packed = scene.pack()
    ds = getattr(scene, "_pgg_device_scene", None)
    if ds is None or ds.device != device or ds.key != packed[0].tobytes():
        ds = DeviceScene(scene, device, packed)
        try:
            scene._pgg_device_scene = ds
        except AttributeError:
            pass
    return ds


def camera_abi(cam):
    c = _lib.Camera()
    for name in ("origin", "forward", "right", "up"):
        v = getattr(cam, name)
        arr = getattr(c, name)
        for i in range(3):
            arr[i] = float(v[i])
    c.tan_half_fov = float(cam.tan_half_fov)
    return c


@dataclass
class FrameGBuffer:
    """Packed G-buffer planes + int32 material ids (-1 on a miss)."""

    planes: GBufferPlanes
    mat: torch.Tensor


def gbuffer_planes(dscene: DeviceScene, cam, width, height, prev_cam=None, row0=0, rows=None,
                   out: Optional[FrameGBuffer] = None, stream=None) -> FrameGBuffer:
    """Primary hits of rows [row0, row0 + rows); prev_cam adds motion vectors
    and has_history (motion_vectors of pg/ptrace.py:132-150)."""
    rows = int(height - row0 if rows is None else rows)
    if out is None:
        out = FrameGBuffer(GBufferPlanes.empty(rows, width, dscene.device, row0=row0),
                           torch.empty(rows, width, dtype=torch.int32, device=dscene.device))
    g = out.planes
    g.cam_origin = tuple(float(c) for c in cam.origin)
    g.height = int(height)
    ca = camera_abi(cam)
    pa = camera_abi(prev_cam) if prev_cam is not None else None
    _lib.check(_lib.lib().pgg_gbuffer_pass(
        ctypes.byref(dscene.abi), ctypes.byref(ca), ctypes.byref(pa) if pa is not None else None, int(width), int(height),
        int(row0), rows, _lib.ptr(g.flags), _lib.ptr(g.nd), _lib.ptr(g.pr), _lib.ptr(g.va), _lib.ptr(g.am),
        _lib.ptr(out.mat), _lib.stream_ptr(stream)))
    return out


@dataclass
class RenderPlanes:
    image: torch.Tensor                  # (rows, W, 3) float32
    vpl: VplPlanes                       # y (pos, usable), L (radiance, valid | strategy << 1)
    lum: Optional[torch.Tensor] = None   # (rows, W, 2) float64 luminance sum, sum of squares
    counters: Optional[torch.Tensor] = None  # int64 [segments, nonfinite]

    @property
    def vpl_valid(self):
        return (self.vpl.L[..., 3].to(torch.int32) & 1).bool()

    @property
    def vpl_strategy(self):
        return (self.vpl.L[..., 3].to(torch.int32) >> 1).to(torch.uint8)


def render_planes(dscene: DeviceScene, fgb: FrameGBuffer, frame, seed, spp=1, max_depth=4, nee=True,
                  depth0: Optional[SamplePlanes] = None, want_moments=False, row0=None, rows=None,
                  out: Optional[RenderPlanes] = None, stream=None, states: Optional[torch.Tensor] = None) -> RenderPlanes:
    """Trace spp lanes per pixel of rows [row0, row0 + rows) (default: the
    G-buffer's rows).  depth0: the guiding pass's samples of the same rows.
    states: caller PCG32 lane states (int64 view, rows*W*spp), advanced in
    place, instead of the (seed, frame, lane) key chain."""
    g = fgb.planes
    W = g.width
    H = int(g.height if g.height is not None else g.row0 + g.rows)
    row0 = g.row0 if row0 is None else int(row0)
    rows = g.row0 + g.rows - row0 if rows is None else int(rows)
    dev = g.flags.device
    if out is None:
        out = RenderPlanes(torch.empty(rows, W, 3, dtype=torch.float32, device=dev),
                           VplPlanes(torch.empty(rows, W, 4, device=dev), torch.empty(rows, W, 4, device=dev),
                                     row0=row0),
                           torch.empty(rows, W, 2, dtype=torch.float64, device=dev) if want_moments else None,
                           torch.zeros(2, dtype=torch.int64, device=dev))
    elif out.counters is not None:
        out.counters.zero_()
    c = _lib.RenderConfig()
    c.width, c.height, c.row0, c.rows = W, H, row0, rows
    c.spp, c.max_depth, c.nee = int(spp), int(max_depth), 1 if nee else 0
    c.key = _lib.frame_key(seed, frame, 0)
    o = _lib.RenderOut(_lib.ptr(out.image), _lib.ptr(out.vpl.y), _lib.ptr(out.vpl.L), _lib.ptr(out.lum),
                       _lib.ptr(out.counters), _lib.ptr(states))
    smp = depth0.as_abi() if depth0 is not None else None
    gabi = g.as_abi()
    _lib.check(_lib.lib().pgg_render_pass(ctypes.byref(c), ctypes.byref(dscene.abi), ctypes.byref(gabi),
                                          _lib.ptr(fgb.mat), ctypes.byref(smp) if smp is not None else None,
                                          ctypes.byref(o), _lib.stream_ptr(stream)))
    return out
