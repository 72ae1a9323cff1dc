"""Multi-frame trajectory of the GPU pass vs the CPU oracle: per-frame
quantiles of the per-channel relative error on Gamma.
Usage: python tools/chain_diag.py [W H FRAMES]"""
import sys
from types import SimpleNamespace

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import pgg_oracle as O  # noqa: E402
from paper_2112_09728_b200 import synth  # noqa: E402
from paper_2112_09728_b200.layout import GBufferPlanes, PassConfig, VplPlanes  # noqa: E402
from paper_2112_09728_b200.session import GuidingSession  # noqa: E402


def ns(d):
    return SimpleNamespace(**{k: (v.numpy().astype(np.float64) if torch.is_tensor(v) and v.dtype == torch.float32
                                  else (v.numpy() if torch.is_tensor(v) else v)) for k, v in d.items()})


def main(w=160, h=120, frames=8, seed=9):
    dev = torch.device("cuda:0")
    sess = GuidingSession(w, h, PassConfig(seed=seed, spp=1), device=dev)
    gam = O.fresh_stats(h * w).reshape(h, w, 8).astype(np.float32)
    prev = None
    for f, (g, v) in enumerate(synth.sequence(w, h, frames, seed=seed)):
        sess.step(GBufferPlanes.from_ref(g, device=dev), VplPlanes.from_ref(v, device=dev), f)
        gn, vn = ns(g), ns(v)
        _, _, gam = O.guiding_frame(gam, prev, gn, vn, seed, f, spp=1)
        prev = gn
        got = sess.gamma.to_aos().cpu().numpy()
        r = np.abs(got.astype(np.float64) - gam) / np.maximum(np.abs(gam.astype(np.float64)), 1e-7)
        worst = np.unravel_index(np.argmax(r), r.shape)
        print(f"frame {f:2d}: frac<=1e-4 {np.mean(r <= 1e-4):.6f} p99 {np.percentile(r, 99):.2e} "
              f"p99.9 {np.percentile(r, 99.9):.2e} max {r.max():.2e} at {worst} k-eq "
              f"{np.mean(got[..., 7] == gam[..., 7]):.6f} per-ch-p99.9 "
              + " ".join(f"{np.percentile(r[..., c], 99.9):.1e}" for c in range(8)), flush=True)


if __name__ == "__main__":
    a = [int(x) for x in sys.argv[1:]]
    main(*a)
