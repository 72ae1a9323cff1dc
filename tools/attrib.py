"""Fixed-input timing of one fused pass at 1080p (for A/B of measurement-only
builds, PGG_LIB=...): the same synthetic G-buffers, VPLs and a random
"trained" Gamma (k uniform in [0, kmax_in]) every time, so stage costs can be
attributed by difference."""

import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kmax-in", type=int, default=16)
    ap.add_argument("--iters", type=int, default=50)
    a = ap.parse_args()
    from paper_2112_09728_b200 import synth
    from paper_2112_09728_b200.layout import GammaPlanes, GBufferPlanes, PassConfig, VplPlanes
    from paper_2112_09728_b200.session import run_pass
    dev = torch.device("cuda:0")
    w, h = 1920, 1080
    (gp, _), (gc, vc) = list(synth.sequence(w, h, 2, seed=1, device=dev, first_frame=7))
    cur = GBufferPlanes.from_ref(gc, device=dev)
    prev = GBufferPlanes.from_ref(gp, device=dev)
    vpl = VplPlanes.from_ref(vc, device=dev)
    g = torch.Generator(device=dev).manual_seed(3)
    st = torch.zeros(h, w, 8, device=dev)
    mu = torch.rand(h, w, 2, device=dev, generator=g) * 0.6 + 0.2
    sd = torch.rand(h, w, 2, device=dev, generator=g) * 0.25 + 0.03
    rho = torch.rand(h, w, device=dev, generator=g) * 1.6 - 0.8
    st[..., 0:2] = mu
    st[..., 2] = sd[..., 0] ** 2 + mu[..., 0] ** 2
    st[..., 3] = sd[..., 1] ** 2 + mu[..., 1] ** 2
    st[..., 4] = rho * sd[..., 0] * sd[..., 1] + mu[..., 0] * mu[..., 1]
    st[..., 6] = torch.rand(h, w, device=dev, generator=g) * 0.9 + 0.05
    st[..., 7] = torch.randint(0, a.kmax_in + 1, (h, w), device=dev, generator=g).float()
    gam = GammaPlanes.from_aos(st, dev)
    cfg = PassConfig(seed=1, spp=1)
    out = GammaPlanes.empty(h, w, dev)
    for _ in range(5):
        run_pass(cfg, 8, cur, gam, prev=prev, vpl=vpl, out_gamma=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        run_pass(cfg, 8, cur, gam, prev=prev, vpl=vpl, out_gamma=out)
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"ms": e0.elapsed_time(e1) / a.iters, "lib": os.environ.get("PGG_LIB", "default"),
                      "kmax_in": a.kmax_in}))


if __name__ == "__main__":
    main()
