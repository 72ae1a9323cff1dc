"""Parity margins of the fused pass on the golden fixtures (Gamma p99.99 /
max relative error per fixture) for the library in PGG_LIB."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import golden_io as gio  # noqa: E402
from paper_2112_09728_b200.layout import GammaPlanes, GBufferPlanes, PassConfig, VplPlanes  # noqa: E402
from paper_2112_09728_b200.session import run_pass  # noqa: E402

dev = torch.device("cuda:0")
out = {"lib": os.environ.get("PGG_LIB", "default")}
z = gio.load("trained_48x40.npz")
spp, seed, fr = int(z["spp"]), int(z["seed"]), int(z["frame"])
cur = GBufferPlanes.from_ref(gio.gbuf_raw(z, "c_"), device=dev)
vpl = VplPlanes.from_ref(gio.vpl_raw(z, "c_"), device=dev)
gin = GammaPlanes.from_aos(z["gamma_in"], dev)
for name, cfg, key in (("trained", PassConfig(seed=seed, spp=spp), "gamma_trained"),
                       ("trained_r7", PassConfig(seed=seed, spp=spp, k_max=32, neighbor_radius=7.3), "gamma_trained_r7")):
    r = run_pass(cfg, fr, cur, gin, vpl=vpl, want_samples=False)
    e = gio.rel_err(r.gamma.to_aos().cpu().numpy(), z[key])
    out[name] = {"p9999": float(np.percentile(e, 99.99)), "max": float(e.max())}
zs = gio.load("seq_64x48.npz")
worst = 0.0
for f in range(6):
    cur = GBufferPlanes.from_ref(gio.gbuf_raw(zs, f"f{f}_"), device=dev)
    r = run_pass(PassConfig(seed=int(zs["seed"]), spp=int(zs["spp"])), f, cur,
                 GammaPlanes.from_aos(zs[f"f{f}_gamma_reproj"], dev),
                 vpl=VplPlanes.from_ref(gio.vpl_raw(zs, f"f{f}_"), device=dev), want_samples=False)
    e = gio.rel_err(r.gamma.to_aos().cpu().numpy(), zs[f"f{f}_gamma_trained"])
    worst = max(worst, float(np.percentile(e, 99.99)))
out["seq_worst_p9999"] = worst
print(json.dumps(out))
