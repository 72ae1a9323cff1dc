"""Small launches of every k_guiding_pass instantiation for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):
  <1,1> TMA VPL tile, VPL planes covering every candidate row (whole frame)
  <1,0> TMA VPL tile, a row band whose VPL planes carry a partial halo
  <0,1> no tile (radius 13 > MAX_TILE_R), whole frame
  <0,0> no tile, partial halo
each with reprojection, 2 spp depth-0 samples and EM, partial edge tiles
(width / height not multiples of the 32 x 8 block), plus the stage-only
entry points.  usage: compute-sanitizer --tool X python tools/sanitize_pass.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2112_09728_b200 import synth  # noqa: E402
from paper_2112_09728_b200.layout import GammaPlanes, GBufferPlanes, PassConfig, VplPlanes  # noqa: E402
from paper_2112_09728_b200.session import run_pass  # noqa: E402

dev = torch.device("cuda:0")
w, h = 100, 70
(gp, _), (gc, vc) = list(synth.sequence(w, h, 2, seed=5, device=dev, first_frame=2))
cur, prev = GBufferPlanes.from_ref(gc, device=dev), GBufferPlanes.from_ref(gp, device=dev)
vfull = VplPlanes.from_ref(vc, device=dev)
gam = GammaPlanes.fresh(h, w, dev)
gam.g1[..., 3] = torch.randint(0, 9, (h, w), device=dev, dtype=torch.float32)
miss = torch.zeros(1, dtype=torch.int32, device=dev)
for radius in (10.0, 13.0):
    cfg = PassConfig(seed=1, spp=2, neighbor_radius=radius)
    # whole frame
    r = run_pass(cfg, 3, cur, gam, prev=prev, vpl=vfull, want_reproj=True, halo_misses=miss)
    # row band [20, 45) with a 4-row VPL halo (partial: < ceil(radius))
    r0, r1, hl = 20, 45, 4
    vb = VplPlanes(vfull.y[r0 - hl:r1 + hl].contiguous(), vfull.L[r0 - hl:r1 + hl].contiguous(), r0 - hl)
    r = run_pass(cfg, 3, cur, gam, prev=prev, vpl=vb, row0=r0, rows=r1 - r0, height=h, want_reproj=True,
                 halo_misses=miss)
    # stage-only calls
    run_pass(cfg, 3, cur, gam, prev=prev, want_reproj=True, want_samples=False)
    run_pass(cfg, 3, cur, gam, want_samples=True)
torch.cuda.synchronize()
print("sanitize_pass ok, halo misses", int(miss.item()))
