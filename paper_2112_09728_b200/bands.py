"""Row-band sharding of the guiding pass over the GPUs of one node
(SURVEY.md 8e): rank r owns the contiguous rows [r0, r1) of the frame; the
only data the pass needs from other ranks are

  * the VPL (Pi) rows within ceil(neighbor_radius) of the band edges, read by
    the EM disk of this frame, and
  * the previous frame's Gamma and G-buffer gate planes (flags, normal+depth)
    within ``max_motion_rows`` of the band edges, read by reprojection.

Every buffer is allocated with its halo rows in place ("extended" buffers,
rows [r0 - h, r1 + h) clipped to the frame); a renderer writes its own band
straight into the middle, and one grouped send/recv (torch.distributed
batch_isend_irecv: NCCL over NVLink on GPUs, gloo in the CPU tests) moves
the boundary rows into the neighbours' halo rows.  RNG streams are keyed on
the GLOBAL pixel index, so any banding reproduces the single-GPU result
bit for bit.
"""

from dataclasses import dataclass

import torch
import torch.distributed as dist


def band_rows(height, world, rank):
    """Balanced contiguous row band of `rank` (first bands get the remainder)."""
    base, rem = divmod(height, world)
    r0 = rank * base + min(rank, rem)
    return r0, r0 + base + (1 if rank < rem else 0)


@dataclass
class Extent:
    """Rows [lo, hi) held by an extended buffer around the band [r0, r1)."""

    r0: int
    r1: int
    lo: int
    hi: int

    @classmethod
    def around(cls, r0, r1, halo, height):
        return cls(r0, r1, max(0, r0 - halo), min(height, r1 + halo))

    @property
    def rows(self):
        return self.hi - self.lo

    def own(self, t):
        """View of the own band inside an extended (rows, ...) tensor."""
        return t[self.r0 - self.lo:self.r1 - self.lo]


def halo_ops(tensors, ext, rank, world, group=None, tag=0):
    """The P2P ops that fill the halo rows of the extended tensors (each
    (ext.rows, W, ...)) from the neighbouring bands: rank-1 sends its last
    rows, rank+1 its first.  Ranks agree on the halo depth, so the rows rank r
    needs from rank r+1 are exactly the rows rank r+1 sends up."""
    ops = []
    if world == 1:
        return ops
    up_rows = ext.r0 - ext.lo       # rows [lo, r0) come from rank - 1
    down_rows = ext.hi - ext.r1     # rows [r1, hi) come from rank + 1
    for t in tensors:
        own = ext.own(t)
        if rank > 0 and up_rows > 0:
            ops.append(dist.P2POp(dist.irecv, t[:up_rows], rank - 1, group, tag))
            ops.append(dist.P2POp(dist.isend, own[:up_rows].contiguous(), rank - 1, group, tag))
        if rank < world - 1 and down_rows > 0:
            ops.append(dist.P2POp(dist.isend, own[own.shape[0] - down_rows:].contiguous(), rank + 1, group, tag))
            ops.append(dist.P2POp(dist.irecv, t[t.shape[0] - down_rows:], rank + 1, group, tag))
    return ops


def post_exchange(ops):
    """Issue one grouped batch of P2P ops; returns the requests (wait() on
    each before reading the halos; on NCCL the wait orders the current CUDA
    stream after the transfer without blocking the host)."""
    return dist.batch_isend_irecv(ops) if ops else []


def halo_exchange(tensors, ext, rank, world, group=None, tag=0):
    """Blocking halo fill of the extended tensors (one grouped batch)."""
    for req in post_exchange(halo_ops(tensors, ext, rank, world, group, tag)):
        req.wait()


def gather_rows(tensors, rank, world, height, group=None):
    """All-gather of every rank's own row band (bands of unequal height are
    padded to the largest) into full-height tensors, in row order."""
    import torch
    base, rem = divmod(height, world)
    mx = base + (1 if rem else 0)
    out = []
    for t in tensors:
        pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[:t.shape[0]] = t
        parts = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad, group=group)  # NCCL on GPUs, gloo in the CPU tests
        full = torch.empty((height,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        for r in range(world):
            r0, r1 = band_rows(height, world, r)
            full[r0:r1] = parts[r][:r1 - r0]
        out.append(full)
    return out


def check_band_geometry(height, world, halo):
    """Every band must be at least `halo` rows tall so that a halo comes from
    the adjacent rank only."""
    for r in range(world):
        r0, r1 = band_rows(height, world, r)
        if r1 - r0 < halo:
            raise ValueError(f"band {r} has {r1 - r0} rows < halo {halo}: too many ranks for this frame height")


class BandedGuiding:
    """One rank's share of a row-band-sharded guiding sequence.

    Per frame: ``frame_inputs()`` hands out the extended buffers to fill (own
    rows only), ``step(frame)`` exchanges halos and runs the fused pass on the
    band.  Gamma, the previous G-buffer and the VPLs live in HBM with their
    halos.  ``max_motion_rows`` bounds |motion_y| + 1 (halo misses are
    counted on the device and reported by ``halo_misses()``)."""

    def __init__(self, width, height, cfg, rank=0, world=1, group=None, device="cuda", max_motion_rows=8):
        from .layout import GammaPlanes, GBufferPlanes, SamplePlanes, VplPlanes
        self.W, self.H, self.cfg = width, height, cfg
        self.rank, self.world, self.group = rank, world, group
        self.dev = torch.device(device)
        r0, r1 = band_rows(height, world, rank)
        self.R = int(-(-cfg.neighbor_radius // 1)) if cfg.neighbor_radius > 0 else 0
        self.M = int(max_motion_rows)
        check_band_geometry(height, world, max(self.R, self.M))
        self.ext_v = Extent.around(r0, r1, self.R, height)   # VPL extent
        self.ext_g = Extent.around(r0, r1, self.M, height)   # Gamma / G-buffer extent
        self.r0, self.r1 = r0, r1
        eg = self.ext_g
        self.gb = [GBufferPlanes.empty(eg.rows, width, self.dev, row0=eg.lo) for _ in range(2)]
        self.gamma = [GammaPlanes.fresh(eg.rows, width, self.dev, row0=eg.lo) for _ in range(2)]
        ev = self.ext_v
        self.vpl = VplPlanes(torch.zeros(ev.rows, width, 4, device=self.dev),
                             torch.zeros(ev.rows, width, 4, device=self.dev), row0=ev.lo)
        self.samples = SamplePlanes.empty(r1 - r0, width, cfg.spp, self.dev)
        self.cur = 0
        self.has_prev = False
        self.prev_gb = None
        self._miss = torch.zeros(1, dtype=torch.int32, device=self.dev)

    def frame_inputs(self):
        """(G-buffer planes, VPL planes) whose OWN rows the caller fills."""
        return self.gb[self.cur], self.vpl

    def extended_planes(self):
        """Fresh (G-buffer, VPL) planes with this band's extents, for callers
        that keep one set per frame and pass them to step()."""
        from .layout import GBufferPlanes, VplPlanes
        eg, ev = self.ext_g, self.ext_v
        gb = GBufferPlanes.empty(eg.rows, self.W, self.dev, row0=eg.lo)
        vp = VplPlanes(torch.zeros(ev.rows, self.W, 4, device=self.dev),
                       torch.zeros(ev.rows, self.W, 4, device=self.dev), row0=ev.lo)
        return gb, vp

    def halo_tensors(self, vpl=None):
        """The (extent, tensors) pairs whose halo rows step() exchanges."""
        vpl = vpl if vpl is not None else self.vpl
        prev = self.prev_gb
        g_in = self.gamma[self.cur]
        pairs = [(self.ext_v, [vpl.y, vpl.L])]
        if self.has_prev:
            pairs.append((self.ext_g, [prev.flags, prev.nd, g_in.g0, g_in.g1]))
        return pairs

    def split_rows(self):
        """(interior, edges): the interior rows of the band read no halo row
        (every read is within max(R, M) rows of the pixel), so they can run
        while the halo exchange is in flight; edges are the rows next to a
        neighbouring band.  Every pixel's result is independent of how the
        band is split into launches (bitwise)."""
        h = max(self.R, self.M)
        lo = self.r0 + (h if self.rank > 0 else 0)
        hi = self.r1 - (h if self.rank < self.world - 1 else 0)
        if hi <= lo:
            return None, [(self.r0, self.r1)]
        edges = [(a, b) for a, b in ((self.r0, lo), (hi, self.r1)) if b > a]
        return (lo, hi), edges

    def _launch(self, frame, a, b, cur_band, vpl, prev, g_in, g_out):
        from .layout import SamplePlanes
        from .session import run_pass
        eg = self.ext_g
        out_view = type(g_out)(g_out.g0[a - eg.lo:b - eg.lo], g_out.g1[a - eg.lo:b - eg.lo], row0=a)
        smp = SamplePlanes(self.samples.dir[a - self.r0:b - self.r0], self.samples.tag[a - self.r0:b - self.r0],
                           self.samples.spp)
        return run_pass(self.cfg, frame, cur_band, g_in, prev=prev if self.has_prev else None, vpl=vpl,
                        height=self.H, row0=a, rows=b - a, out_gamma=out_view, out_samples=smp,
                        halo_misses=self._miss)

    def history_own(self):
        """This band's own rows of what reprojection reads from other bands:
        previous gate planes (flags, normal+depth) and the current Gamma."""
        eg = self.ext_g
        g_in = self.gamma[self.cur]
        prev = self.prev_gb
        return [eg.own(prev.flags), eg.own(prev.nd), eg.own(g_in.g0), eg.own(g_in.g1)]

    def _full_history_rerun(self, frame, cur_band, vpl, g_out, full):
        """Re-run the band with the whole previous frame as reprojection
        source (flags, nd, g0, g1 full-height), for motion beyond the halo."""
        from .layout import GammaPlanes, GBufferPlanes
        from .session import run_pass
        flags, nd, g0, g1 = full
        prev = GBufferPlanes(flags, nd, nd, nd, nd, self.prev_gb.cam_origin, row0=0)  # only flags / nd are read
        gin = GammaPlanes(g0, g1, row0=0)
        eg = self.ext_g
        out_view = type(g_out)(eg.own(g_out.g0), eg.own(g_out.g1), row0=self.r0)
        self._miss.zero_()
        run_pass(self.cfg, frame, cur_band, gin, prev=prev, vpl=vpl, height=self.H, row0=self.r0,
                 rows=self.r1 - self.r0, out_gamma=out_view, out_samples=self.samples, halo_misses=self._miss)

    def step(self, frame, exchange=True, gbuf=None, vpl=None, overlap=True, split=None, fallback=False,
             gather=None, any_miss=None):
        """Exchange halos (unless the caller already filled them, exchange=False)
        and run the fused pass on this band.  ``gbuf``/``vpl``: this frame's
        extended planes (own rows filled); default: the internal buffers.

        overlap=True: the grouped send/recv is posted first, the
        interior rows run while it is in flight, and the edge rows after the
        stream has waited on it; overlap=False runs exchange, then one launch.
        split=True/False forces the interior/edge launches on or off.

        fallback=True handles motion beyond the halo: if any rank
        counted a reprojection halo miss this frame (``any_miss``, default an
        all-reduce MAX), every rank all-gathers the previous frame's gate
        planes and Gamma (``gather``, default gather_rows) and re-runs its
        band with the whole frame as source, which restores the 1-GPU result.
        It costs one host sync per frame."""
        from .session import PassResult
        cur = self.gb[self.cur] if gbuf is None else gbuf
        vpl = vpl if vpl is not None else self.vpl
        prev = self.prev_gb
        g_in, g_out = self.gamma[self.cur], self.gamma[1 - self.cur]
        eg = self.ext_g
        cur_band = type(cur)(eg.own(cur.flags), eg.own(cur.nd), eg.own(cur.pr), eg.own(cur.va), eg.own(cur.am),
                             cur.cam_origin, row0=self.r0)
        reqs = []
        if exchange and self.world > 1:
            # halos: this frame's VPLs; previous frame's Gamma and gate planes
            ops = []
            for tag, (ext, ts) in enumerate(self.halo_tensors(vpl)):
                ops += halo_ops(ts, ext, self.rank, self.world, self.group, tag=1 + tag)
            reqs = post_exchange(ops)
        if fallback:
            self._miss.zero_()
        if split is None:
            split = overlap and bool(reqs)
        interior, edges = self.split_rows() if split else (None, [(self.r0, self.r1)])
        if interior is not None:
            self._launch(frame, *interior, cur_band, vpl, prev, g_in, g_out)
        for req in reqs:
            req.wait()
        for a, b in edges:
            self._launch(frame, a, b, cur_band, vpl, prev, g_in, g_out)
        if fallback and self.has_prev:
            if any_miss is None:
                import torch
                m = self._miss.clone().to(torch.int64)
                if self.world > 1:
                    dist.all_reduce(m, op=dist.ReduceOp.MAX, group=self.group)
                missed = int(m.item()) > 0
            else:
                missed = bool(any_miss(int(self._miss.item())))
            if missed:
                own = self.history_own()
                full = gather(own) if gather is not None else gather_rows(own, self.rank, self.world, self.H,
                                                                           self.group)
                self._full_history_rerun(frame, cur_band, vpl, g_out, full)
        self.cur = 1 - self.cur
        self.has_prev = True
        self.prev_gb = cur
        from .layout import GammaPlanes
        return PassResult(gamma=GammaPlanes(eg.own(g_out.g0), eg.own(g_out.g1), row0=self.r0), samples=self.samples)

    @property
    def gamma_own(self):
        """This rank's band of the latest Gamma (planes views)."""
        g = self.gamma[self.cur]
        return self.ext_g.own(g.g0), self.ext_g.own(g.g1)

    def halo_misses(self):
        return int(self._miss.item())
