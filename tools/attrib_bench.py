"""Stage attribution on the bench workload's own state: `--save P` runs the
1080p bench sequence for F frames with the product library and saves Gamma;
`--load P` (with PGG_LIB = a measurement-only build) times the fused pass of
frame F on that fixed state (CUDA events, median of --iters launches)."""
import argparse
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--save")
    ap.add_argument("--load")
    ap.add_argument("--frames", type=int, default=8)
    ap.add_argument("--iters", type=int, default=40)
    a = ap.parse_args()
    from paper_2112_09728_b200 import synth
    from paper_2112_09728_b200.layout import GammaPlanes, GBufferPlanes, PassConfig, VplPlanes
    from paper_2112_09728_b200.session import GuidingSession, run_pass
    dev = torch.device("cuda:0")
    w, h, F = 1920, 1080, a.frames
    frames = [(GBufferPlanes.from_ref(g, device=dev), VplPlanes.from_ref(v, device=dev))
              for g, v in synth.sequence(w, h, F + 1, seed=0, device=dev)]
    cfg = PassConfig(seed=0, spp=1)
    if a.save:
        sess = GuidingSession(w, h, cfg, device=dev)
        for f in range(F):
            sess.step(frames[f][0], frames[f][1], f)
        torch.save({"g0": sess.gamma.g0.cpu(), "g1": sess.gamma.g1.cpu()}, a.save)
        return
    d = torch.load(a.load)
    gam = GammaPlanes(d["g0"].to(dev), d["g1"].to(dev))
    out = GammaPlanes.empty(h, w, dev)
    r = None
    for _ in range(5):
        r = run_pass(cfg, F, frames[F][0], gam, prev=frames[F - 1][0], vpl=frames[F][1], out_gamma=out)
    ts = []
    for _ in range(a.iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run_pass(cfg, F, frames[F][0], gam, prev=frames[F - 1][0], vpl=frames[F][1], out_gamma=out,
                 out_samples=r.samples)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(json.dumps({"ms": statistics.median(ts), "lib": os.environ.get("PGG_LIB", "default"), "frame": F}))


if __name__ == "__main__":
    main()
