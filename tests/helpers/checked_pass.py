"""Run by tests/test_gpu_checked.py in a fresh process, with PGG_LIB pointing
at libpgg_checked.so (in-kernel bounds asserts) or at the product library.

Every k_guiding_pass instantiation -- TMA tile / global VPLs x whole-frame /
partial-halo VPL planes -- on frames whose size is not a multiple of the
32 x 8 block, with reprojection, 2 spp samples and EM, plus the stage-only
calls.  Outputs live inside larger allocations whose guard rows are filled
with a sentinel and the outputs themselves pre-filled with NaN: afterwards
every output element of the launch's band must have been written (no NaN,
i.e. no read of an unwritten output, no skipped pixel) and every guard word
must be untouched (no out-of-band write).  Prints one JSON line."""
import ctypes
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2112_09728_b200 import _lib, synth  # noqa: E402
from paper_2112_09728_b200.layout import GammaPlanes, GBufferPlanes, PassConfig, SamplePlanes, VplPlanes  # noqa: E402
from paper_2112_09728_b200.session import run_pass  # noqa: E402

SENT = -7.25e30
GUARD = 3
dev = torch.device("cuda:0")
out = {"lib": _lib.LIB_PATH, "launches": 0, "unwritten": 0, "guard_overwrites": 0}


def guarded(rows, w, spp):
    """(planes view, guard tensors) with GUARD sentinel rows on both sides"""
    g0 = torch.full((rows + 2 * GUARD, w, 4), SENT, device=dev)
    g1 = torch.full((rows + 2 * GUARD, w, 4), SENT, device=dev)
    d = torch.full((rows + 2 * GUARD, w, spp, 4), SENT, device=dev)
    t = torch.full((rows + 2 * GUARD, w, spp), 0xAB, dtype=torch.uint8, device=dev)
    mid = slice(GUARD, GUARD + rows)
    for x in (g0, g1, d):
        x[mid] = float("nan")
    t[mid] = 0xCD
    gam = GammaPlanes(g0[mid], g1[mid])
    smp = SamplePlanes(d[mid], t[mid])
    return gam, smp, (g0, g1, d, t)


def verify(full, rows, with_gamma=True, with_smp=True):
    g0, g1, d, t = full
    mid = slice(GUARD, GUARD + rows)
    out["launches"] += 1
    for x, used in ((g0, with_gamma), (g1, with_gamma), (d, with_smp)):
        for side in (x[:GUARD], x[GUARD + rows:]):
            out["guard_overwrites"] += int((side != SENT).sum().item())
        if used:
            out["unwritten"] += int(torch.isnan(x[mid]).sum().item())
    for side in (t[:GUARD], t[GUARD + rows:]):
        out["guard_overwrites"] += int((side != 0xAB).sum().item())
    if with_smp:
        out["unwritten"] += int((t[mid] == 0xCD).sum().item())


for w, h in ((100, 70), (37, 29), (256, 64)):
    (gp, _), (gc, vc) = list(synth.sequence(w, h, 2, seed=5, device=dev, first_frame=2))
    cur, prev = GBufferPlanes.from_ref(gc, device=dev), GBufferPlanes.from_ref(gp, device=dev)
    vfull = VplPlanes.from_ref(vc, device=dev)
    gam = GammaPlanes.fresh(h, w, dev)
    gam.g1[..., 3] = torch.randint(0, 9, (h, w), device=dev, dtype=torch.float32)
    miss = torch.zeros(1, dtype=torch.int32, device=dev)
    for radius in (10.0, 12.0, 13.0, 7.3):
        cfg = PassConfig(seed=1, spp=2, neighbor_radius=radius)
        bands = [(0, h, None)]
        if h > 40:
            bands += [(20, 45, 4), (0, 25, 30), (h - 21, h, 2)]   # partial halo, full halo, frame edge
        for r0, r1, hl in bands:
            rows = r1 - r0
            if hl is None:
                vp = vfull
            else:
                lo, hi = max(0, r0 - hl), min(h, r1 + hl)
                vp = VplPlanes(vfull.y[lo:hi].contiguous(), vfull.L[lo:hi].contiguous(), lo)
            go, so, full = guarded(rows, w, 2)
            gr, _, full_r = guarded(rows, w, 2)
            run_pass(cfg, 3, cur, gam, prev=prev, vpl=vp, row0=r0, rows=rows, height=h, want_reproj=True,
                     out_gamma=go, out_reproj=gr, out_samples=so, halo_misses=miss)
            torch.cuda.synchronize()
            verify(full, rows)
            verify(full_r, rows, with_smp=False)
            # training alone: the EM-only instantiations (kStage 2)
            go2, _, full2 = guarded(rows, w, 2)
            run_pass(cfg, 3, cur, gam, vpl=vp, row0=r0, rows=rows, height=h, want_samples=False, out_gamma=go2,
                     halo_misses=miss)
            torch.cuda.synchronize()
            verify(full2, rows, with_smp=False)
        # stage-only calls
        gr, _, full_r = guarded(h, w, 2)
        run_pass(cfg, 3, cur, gam, prev=prev, want_reproj=True, want_samples=False, out_reproj=gr)
        torch.cuda.synchronize()
        verify(full_r, h, with_smp=False)
        _, so, full = guarded(h, w, 2)
        run_pass(cfg, 3, cur, gam, want_samples=True, out_samples=so)
        torch.cuda.synchronize()
        verify(full, h, with_gamma=False)
out["halo_misses"] = int(miss.item())
chk = (ctypes.c_int32 * 6)()
rc = _lib.lib().pgg_debug_checks(chk, 1)
out["checked_build"] = rc == 0
out["check_failures"] = int(chk[0]) if rc == 0 else None
out["first_failure"] = list(chk)[1:] if rc == 0 and chk[0] else None
print(json.dumps(out))
