"""Screen-space guiding state and its GPU passes; drop-in for
pgtrace.guide_buffers (pg/guide_buffers.py).

``reproject`` and ``training_pass`` keep the reference's signatures and
double-buffered semantics (they return a new GuidingBuffer with
generation + 1) and run the fused libpgg kernel on the device.
``guiding_frame`` is the fused one-launch form of reproject -> depth-0
sampling -> training that a GPU renderer should call instead.
``GuidingBuffer.stats`` may be a NumPy (H,W,8) float32 array (reference
behaviour, host round trip per call) or a CUDA tensor (stays resident).
"""

import dataclasses
import struct
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np
import torch

from . import _conv, _lib, mixture
from .layout import GammaPlanes, GBufferPlanes, PassConfig, SamplePlanes, VplPlanes
from .session import run_pass

CHECKPOINT_MAGIC = b"PGG1"
NEIGHBOR_RADIUS = 10.0
_MAX_CANDIDATES = 20

# access instrumentation (pg/guide_buffers.py:22-38)
_access_count = 0


def note_access():
    global _access_count
    _access_count += 1


def access_count():
    return _access_count


def reset_access_count():
    global _access_count
    _access_count = 0


class CheckpointError(ValueError):
    """Raised for malformed or mismatched checkpoint files."""


@dataclass
class GuidingBuffer:
    """Gamma: (H, W, 8) float32 per-pixel mixture state (pg/guide_buffers.py:45-59)."""

    width: int
    height: int
    stats: object
    generation: int = 0

    @classmethod
    def create(cls, width, height, device=None):
        """init_stats everywhere; ``device="cuda"`` keeps it on the GPU."""
        g = GammaPlanes.fresh(height, width, _conv.device()).to_aos()
        return cls(width, height, g if device is not None else g.cpu().numpy())

    def stats_for_render(self):
        note_access()
        if torch.is_tensor(self.stats):
            return self.stats.to(torch.float64)
        return np.asarray(self.stats).astype(np.float64)

    def planes(self):
        return GammaPlanes.from_aos(self.stats, _conv.device())


@dataclass
class ReprojectionPolicy:
    depth_rel_tol: float = 0.1
    normal_dot_min: float = 0.9
    rotate_mean: bool = True


class RadianceSampleRec(NamedTuple):
    """One training record (pg/guide_buffers.py:69-75)."""

    sq: np.ndarray
    direction: np.ndarray
    weight: float
    strategy: int


def _planes(g):
    """Device planes of any GuidingBuffer-like object (ours or the
    reference's pgtrace.guide_buffers.GuidingBuffer: width, height, stats)."""
    return GammaPlanes.from_aos(g.stats, _conv.device())


def _wrap(stats_tensor, like, generation):
    """A new buffer of the caller's own GuidingBuffer class (the reference's
    dataclass when a pgtrace session calls us), stats as NumPy or as the
    caller's CUDA tensor type -- double buffering, generation + 1
    (pg/guide_buffers.py:135-137, 281-283)."""
    st = stats_tensor if torch.is_tensor(like.stats) else stats_tensor.cpu().numpy()
    if dataclasses.is_dataclass(like):
        return dataclasses.replace(like, stats=st, generation=generation)
    return GuidingBuffer(like.width, like.height, st, generation)


def reproject(gamma_prev, gbuf_prev, gbuf_cur, policy):
    """Nearest-neighbour history fetch along motion vectors with depth /
    normal rejection and mean rotation (pg/guide_buffers.py:78-137)."""
    note_access()
    dev = _conv.device()
    h, w = gamma_prev.height, gamma_prev.width
    cur = GBufferPlanes.from_ref(gbuf_cur, device=dev)
    prev = GBufferPlanes.from_ref(gbuf_prev, device=dev)
    cfg = PassConfig(depth_rel_tol=policy.depth_rel_tol, normal_dot_min=policy.normal_dot_min,
                     rotate_mean=policy.rotate_mean)
    miss = torch.zeros(1, dtype=torch.int32, device=dev)
    res = run_pass(cfg, 0, cur, _planes(gamma_prev), prev=prev, height=h, want_reproj=True, want_samples=False,
                   halo_misses=miss)
    return _wrap(res.gamma_reproj.to_aos(), gamma_prev, gamma_prev.generation + 1)


def training_pass(gamma, vpl, gbuf, k_max=mixture.KMAX_DEFAULT, seed=0, frame_index=0,
                  neighbor_radius=NEIGHBOR_RADIUS):
    """One EM epoch per valid pixel over the screen-space VPL disk
    (pg/guide_buffers.py:262-283)."""
    note_access()
    dev = _conv.device()
    h, w = gamma.height, gamma.width
    cfg = PassConfig(seed=seed, k_max=k_max, neighbor_radius=neighbor_radius)
    res = run_pass(cfg, frame_index, GBufferPlanes.from_ref(gbuf, device=dev), _planes(gamma),
                   vpl=VplPlanes.from_ref(vpl, device=dev), height=h, want_samples=False)
    return _wrap(res.gamma.to_aos(), gamma, gamma.generation + 1)


def guiding_frame(gamma_prev, gbuf_prev, gbuf, vpl, seed=0, frame_index=0, spp=1, nee_draws=3,
                  k_max=mixture.KMAX_DEFAULT, neighbor_radius=NEIGHBOR_RADIUS, policy=None,
                  roughness_min_guide=0.05):
    """The whole guiding pass of one frame in ONE kernel launch:
    reproject (when gbuf_prev is given) -> depth-0 guided sampling -> EM
    (pg/cli.py:114-142 order).  Returns (gamma_reproj, samples dict, gamma_trained)."""
    note_access()
    dev = _conv.device()
    policy = policy or ReprojectionPolicy()
    h, w = gamma_prev.height, gamma_prev.width
    cfg = PassConfig(seed=seed, spp=spp, nee_draws=nee_draws, k_max=k_max, neighbor_radius=neighbor_radius,
                     depth_rel_tol=policy.depth_rel_tol, normal_dot_min=policy.normal_dot_min,
                     rotate_mean=policy.rotate_mean, roughness_min_guide=roughness_min_guide)
    prev = GBufferPlanes.from_ref(gbuf_prev, device=dev) if gbuf_prev is not None else None
    res = run_pass(cfg, frame_index, GBufferPlanes.from_ref(gbuf, device=dev), _planes(gamma_prev), prev=prev,
                   vpl=VplPlanes.from_ref(vpl, device=dev), height=h, want_reproj=True, want_samples=True)
    d = res.samples.dir.reshape(h * w, spp, 4)
    t = res.samples.tag.reshape(h * w, spp)
    smp = dict(wi=d[..., :3].to(torch.float64), pdf=d[..., 3].to(torch.float64), strategy=t & 1,
               valid=((t >> 1) & 1).bool())
    if not torch.is_tensor(gamma_prev.stats):
        smp = {k: v.cpu().numpy() for k, v in smp.items()}
    g_rep = _wrap(res.gamma_reproj.to_aos(), gamma_prev, gamma_prev.generation + 1)
    g_tr = _wrap(res.gamma.to_aos(), gamma_prev, gamma_prev.generation + 2)
    return g_rep, smp, g_tr


# ---------------------------------------------------------------------------
# checkpoints: magic, u32 width/height, row-major float32 LE stats
# (pg/guide_buffers.py:289-314)

def checkpoint_save(gamma, path):
    st = gamma.stats.detach().cpu().numpy() if torch.is_tensor(gamma.stats) else np.asarray(gamma.stats)
    with open(path, "wb") as f:
        f.write(CHECKPOINT_MAGIC)
        f.write(struct.pack("<II", gamma.width, gamma.height))
        f.write(np.ascontiguousarray(st, dtype="<f4").tobytes())


def checkpoint_load(path, expect_size=None, device=None):
    """Load a stats checkpoint; optionally enforce (width, height);
    ``device="cuda"`` returns a device-resident GuidingBuffer."""
    with open(path, "rb") as f:
        magic = f.read(4)
        if magic != CHECKPOINT_MAGIC:
            raise CheckpointError(f"bad checkpoint magic {magic!r} (version mismatch?)")
        header = f.read(8)
        if len(header) != 8:
            raise CheckpointError("truncated checkpoint header")
        w, h = struct.unpack("<II", header)
        if expect_size is not None and (w, h) != tuple(expect_size):
            raise CheckpointError(f"checkpoint is {w}x{h}, session expects {expect_size[0]}x{expect_size[1]}")
        payload = f.read(w * h * 8 * 4)
        if len(payload) != w * h * 8 * 4:
            raise CheckpointError("truncated checkpoint payload")
        stats = np.frombuffer(payload, dtype="<f4").reshape(h, w, 8).copy()
    if device is not None:
        return GuidingBuffer(w, h, torch.from_numpy(stats).to(device))
    return GuidingBuffer(w, h, stats)


def gather_training_batch(pixel_xy, vpl, gbuf, gamma, k_max, streams):
    """Training records of one pixel, self VPL first (pg/guide_buffers.py:234-259).

    ``streams`` holds one PCG32 state per buffer pixel; like the reference,
    every stream is advanced by the 38 candidate draws of the pass."""
    from . import rng, sgmap
    note_access()
    dev = _conv.device()
    x, y = (int(v) for v in pixel_xy)
    h, w = gbuf.height, gbuf.width
    cur = GBufferPlanes.from_ref(gbuf, device=dev)
    vp = VplPlanes.from_ref(vpl, device=dev)
    gp = _planes(gamma)
    st = _conv.u64_to_dev(streams).reshape(-1)
    cfg = PassConfig(k_max=k_max, neighbor_radius=NEIGHBOR_RADIUS)
    from .layout import make_config
    c = make_config(cfg, w, h, 0)
    px = torch.tensor([[x, y]], dtype=torch.int32, device=dev)
    rec = torch.empty(1, _MAX_CANDIDATES, 4, dtype=torch.float32, device=dev)
    import ctypes
    ref = ctypes.byref
    cur_abi, gin, vabi = cur.as_abi(), gp.as_in(), vp.as_abi()
    _lib.check(_lib.lib().pgg_train_records(ref(c), ref(cur_abi), ref(gin), ref(vabi), 1, _lib.ptr(px), _lib.ptr(st),
                                            _lib.ptr(rec), _lib.stream_ptr()))
    # the reference's pass draws 2 x 19 numbers from every stream
    for _ in range(2 * (_MAX_CANDIDATES - 1)):
        rng.next_u32(st)
    if torch.is_tensor(streams):
        streams.view(torch.int64).copy_(st.view(streams.shape))
    else:
        np.asarray(streams)[...] = st.cpu().numpy().view(np.uint64).reshape(np.asarray(streams).shape)
    r = rec[0].to(torch.float64)
    n = _conv.to_dev(np.asarray(gbuf.normal).reshape(-1, 3)[y * w + x] if not torch.is_tensor(gbuf.normal)
                     else gbuf.normal.reshape(-1, 3)[y * w + x], torch.float64)
    t, b = sgmap.build_tangent_frame(n)
    out = []
    for slot in range(_MAX_CANDIDATES):
        if r[slot, 3] > 0:
            sq = r[slot, :2]
            d = sgmap.to_world(t, b, n, sgmap.square_to_hemisphere(sq))
            out.append(RadianceSampleRec(sq.cpu().numpy(), d.cpu().numpy(), float(r[slot, 2]), mixture.STRATEGY_BRDF))
    return out
