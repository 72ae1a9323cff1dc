"""Bitwise equality of two builds of the pass (e.g. the fused kernel and the
stage-split launches): runs the bench sequence's frames through both
libraries in two processes and compares Gamma', the reprojected Gamma and the
samples.  Usage: python tools/split_equal.py libA.so libB.so"""
import os
import subprocess
import sys

import numpy as np

if len(sys.argv) == 3 and sys.argv[2] != "--child":
    outs = []
    for lib in sys.argv[1:]:
        path = f"/tmp/split_eq_{os.path.basename(lib)}.npz"
        subprocess.run([sys.executable, __file__, path, "--child"], check=True, env={**os.environ, "PGG_LIB": lib})
        outs.append(np.load(path))
    bad = [k for k in outs[0].files if not np.array_equal(outs[0][k], outs[1][k])]
    print("bitwise equal" if not bad else f"DIFFER: {bad}", {k: outs[0][k].shape for k in outs[0].files})
    sys.exit(1 if bad else 0)

import torch  # noqa: E402

sys.path.insert(0, ".")
from paper_2112_09728_b200 import synth  # noqa: E402
from paper_2112_09728_b200.layout import GammaPlanes, GBufferPlanes, PassConfig, VplPlanes  # noqa: E402
from paper_2112_09728_b200.session import run_pass  # noqa: E402

dev = torch.device("cuda:0")
w, h = 1920, 1080
res = {}
for spp in (1, 2):
    cfg = PassConfig(seed=4, spp=spp)
    frames = [(GBufferPlanes.from_ref(g, device=dev), VplPlanes.from_ref(v, device=dev))
              for g, v in synth.sequence(w, h, 6, seed=4, device=dev)]
    gam = GammaPlanes.fresh(h, w, dev)
    for f, (cur, vp) in enumerate(frames):
        r = run_pass(cfg, f, cur, gam, prev=frames[f - 1][0] if f else None, vpl=vp, want_reproj=f > 0)
        gam = r.gamma
    res[f"gamma_{spp}"] = gam.to_aos().cpu().numpy()
    res[f"reproj_{spp}"] = r.gamma_reproj.to_aos().cpu().numpy()
    res[f"dir_{spp}"] = r.samples.dir.cpu().numpy()
    res[f"tag_{spp}"] = r.samples.tag.cpu().numpy()
    # training only and sampling only (the single-stage entry points)
    t = run_pass(cfg, 6, frames[5][0], gam, vpl=frames[5][1], want_samples=False)
    res[f"train_{spp}"] = t.gamma.to_aos().cpu().numpy()
    s = run_pass(cfg, 6, frames[5][0], gam, prev=frames[4][0])
    res[f"smp_only_{spp}"] = s.samples.dir.cpu().numpy()
np.savez(sys.argv[1], **res)
