"""Worst depth-0 direction errors of the 4K 4 spp pass vs the oracle (the
test_4k_4spp_vs_oracle bands): lane, strategy, material, roughness, error."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from oracle import pgg_oracle as O  # noqa: E402
from paper_2112_09728_b200 import synth  # noqa: E402
from paper_2112_09728_b200.layout import GammaPlanes, GBufferPlanes, PassConfig, VplPlanes  # noqa: E402
from paper_2112_09728_b200.session import GuidingSession, run_pass  # noqa: E402
from test_gpu_pass import _ns, _samples  # noqa: E402

dev = torch.device("cuda:0")
w, h, seed, spp, F = 3840, 2160, 0, 4, 5
frames = list(synth.sequence(w, h, F, seed=seed, device=dev))
cfg = PassConfig(seed=seed, spp=spp)
sess = GuidingSession(w, h, cfg, device=dev)
for f in range(F - 1):
    g, v = frames[f]
    sess.step(GBufferPlanes.from_ref(g, device=dev), VplPlanes.from_ref(v, device=dev), f)
gin = sess.gamma.to_aos().cpu().numpy()
(gp, _), (gc, vc) = frames[F - 2], frames[F - 1]
r = run_pass(cfg, F - 1, GBufferPlanes.from_ref(gc, device=dev), GammaPlanes.from_aos(gin, dev),
             prev=GBufferPlanes.from_ref(gp, device=dev), vpl=VplPlanes.from_ref(vc, device=dev))
smp = _samples(r, w * h, spp)
gpn, gcn, vcn = _ns(gp), _ns(gc), _ns(vc)
out = []
for r0, r1 in ((0, 16), (1072, 1088), (2144, 2160)):
    _, osmp, otr = O.guiding_frame(gin, gpn, gcn, vcn, seed, F - 1, spp=spp, rows=(r0, r1))
    band = slice(r0 * w, r1 * w)
    e = np.abs(smp["wi"][band] - osmp["wi"]).max(-1)
    idx = np.argsort(e.ravel())[::-1][:8]
    for i in idx:
        p, s = divmod(int(i), spp)
        y, x = r0 + p // w, p % w
        out.append(dict(band=[r0, r1], y=y, x=x, lane=s, err=float(e.ravel()[i]),
                        strategy=int(osmp["strategy"][p, s]), valid=bool(osmp["valid"][p, s]),
                        kind=int(gcn.kind[y, x]), rough=float(gcn.roughness[y, x]),
                        wi_gpu=smp["wi"][band][p, s].tolist(), wi_ref=osmp["wi"][p, s].tolist(),
                        pdf_gpu=float(smp["pdf"][band][p, s]), pdf_ref=float(osmp["pdf"][p, s])))
    print(json.dumps({"band": [r0, r1], "max": float(e.max()), "n_gt_1e5": int((e > 1e-5).sum()),
                      "n_gt_3e6": int((e > 3e-6).sum())}), flush=True)
for o in out:
    print(json.dumps(o))
