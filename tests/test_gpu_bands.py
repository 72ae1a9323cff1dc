"""Row-band sharding on ONE GPU: N BandedGuiding ranks, halos filled by a
local copy standing in for the NCCL exchange, must reproduce the
whole-frame session bit for bit over a multi-frame sequence (SURVEY 8e:
outputs at N GPUs bitwise equal to 1 GPU)."""

import pytest
import torch

pytestmark = pytest.mark.gpu


def _fill(band, g, v):
    """Write a band's OWN rows of frame inputs (as a renderer of that band would)."""
    from paper_2112_09728_b200.layout import GBufferPlanes, VplPlanes
    gb, vp = band.frame_inputs()
    full_g = GBufferPlanes.from_ref(g, device=band.dev)
    full_v = VplPlanes.from_ref(v, device=band.dev)
    r0, r1 = band.r0, band.r1
    for name in ("flags", "nd", "pr", "va", "am"):
        band.ext_g.own(getattr(gb, name)).copy_(getattr(full_g, name)[r0:r1])
    gb.cam_origin = full_g.cam_origin
    band.ext_v.own(vp.y).copy_(full_v.y[r0:r1])
    band.ext_v.own(vp.L).copy_(full_v.L[r0:r1])


def _local_exchange(bands):
    """What halo_exchange does over NCCL: halo rows <- neighbours' own rows."""
    for b in bands:
        for k, (ext, ts) in enumerate(b.halo_tensors()):
            for t_i, t in enumerate(ts):
                for nb in bands:
                    if nb is b:
                        continue
                    next_, nts = nb.halo_tensors()[k]
                    src = nts[t_i]
                    lo, hi = max(ext.lo, nb.r0), min(ext.hi, nb.r1)
                    if lo < hi:
                        t[lo - ext.lo:hi - ext.lo].copy_(src[lo - next_.lo:hi - next_.lo])


@pytest.mark.parametrize("world,split", [(2, False), (3, False), (5, False), (2, True), (3, True)])
def test_bands_match_whole_frame(cuda_dev, world, split):
    """split=True: interior rows and edge rows in separate launches, as in the
    overlapped exchange path."""
    from paper_2112_09728_b200 import synth
    from paper_2112_09728_b200.bands import BandedGuiding
    from paper_2112_09728_b200.layout import GBufferPlanes, PassConfig, VplPlanes
    from paper_2112_09728_b200.session import GuidingSession
    W, H, F, seed = 320, 184, 4, 11
    cfg = PassConfig(seed=seed, spp=2)
    frames = list(synth.sequence(W, H, F, seed=seed, device=cuda_dev))
    whole = GuidingSession(W, H, cfg, device=cuda_dev)
    bands = [BandedGuiding(W, H, cfg, rank=r, world=world, device=cuda_dev, max_motion_rows=8) for r in range(world)]
    for f, (g, v) in enumerate(frames):
        ref = whole.step(GBufferPlanes.from_ref(g, device=cuda_dev), VplPlanes.from_ref(v, device=cuda_dev), f)
        for b in bands:
            _fill(b, g, v)
        _local_exchange(bands)
        for b in bands:
            b.step(f, exchange=False, split=split)
        torch.cuda.synchronize()
        g0 = torch.cat([b.gamma_own[0] for b in bands])
        g1 = torch.cat([b.gamma_own[1] for b in bands])
        assert torch.equal(g0, whole.gamma.g0) and torch.equal(g1, whole.gamma.g1), f
        sd = torch.cat([b.samples.dir for b in bands])
        st = torch.cat([b.samples.tag for b in bands])
        assert torch.equal(sd, whole.samples.dir) and torch.equal(st, whole.samples.tag), f
    assert all(b.halo_misses() == 0 for b in bands)


def test_large_motion_full_history_fallback(cuda_dev):
    """Vertical motion beyond the reprojection halo: the bands count misses,
    and the full-history fallback (all-gather of the previous gate planes and
    Gamma, here assembled locally) restores the whole-frame result bit for bit."""
    from paper_2112_09728_b200 import synth
    from paper_2112_09728_b200.bands import BandedGuiding
    from paper_2112_09728_b200.layout import GBufferPlanes, PassConfig, VplPlanes
    from paper_2112_09728_b200.session import GuidingSession
    W, H, F, seed, world = 256, 120, 3, 6, 3
    cfg = PassConfig(seed=seed, spp=1)
    frames = []
    for f, (g, v) in enumerate(synth.sequence(W, H, F, seed=seed, device=cuda_dev)):
        g = dict(g)
        if f > 0:
            g["motion"] = g["motion"].clone()
            g["motion"][..., 1] += 5.0  # 5-6 rows of vertical motion
        frames.append((g, v))
    whole = GuidingSession(W, H, cfg, device=cuda_dev)
    bands = [BandedGuiding(W, H, cfg, rank=r, world=world, device=cuda_dev, max_motion_rows=2) for r in range(world)]
    plain = [BandedGuiding(W, H, cfg, rank=r, world=world, device=cuda_dev, max_motion_rows=2) for r in range(world)]
    for f, (g, v) in enumerate(frames):
        whole.step(GBufferPlanes.from_ref(g, device=cuda_dev), VplPlanes.from_ref(v, device=cuda_dev), f)
        for bs in (bands, plain):
            for b in bs:
                _fill(b, g, v)
            _local_exchange(bs)
        hist = [[t.clone() for t in b.history_own()] for b in bands] if bands[0].has_prev else None
        gather = (lambda own: [torch.cat([h[k] for h in hist]) for k in range(4)]) if hist else None
        for b in bands:
            b.step(f, exchange=False, fallback=True, gather=gather, any_miss=lambda m: m > 0)
        for b in plain:
            b.step(f, exchange=False)
        torch.cuda.synchronize()
        g0 = torch.cat([b.gamma_own[0] for b in bands])
        g1 = torch.cat([b.gamma_own[1] for b in bands])
        assert torch.equal(g0, whole.gamma.g0) and torch.equal(g1, whole.gamma.g1), f
    assert sum(b.halo_misses() for b in plain) > 0  # the halo really was too small
    p0 = torch.cat([b.gamma_own[0] for b in plain])
    assert not torch.equal(p0, whole.gamma.g0)
