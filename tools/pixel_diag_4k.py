"""One pixel of the 4K 4 spp pass (tools/dir_worst_4k.py's worst lane):
input Gamma, reprojected Gamma GPU vs oracle, lobe, the oracle's draws."""
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

Y, X = int(sys.argv[1]), int(sys.argv[2])
SEED = int(sys.argv[3]) if len(sys.argv) > 3 else 0
FR = int(sys.argv[4]) if len(sys.argv) > 4 else 5
np.set_printoptions(precision=12, linewidth=160)
dev = torch.device("cuda:0")
w, h, seed, spp, F = 3840, 2160, SEED, 4, FR
frames = list(synth.sequence(w, h, F, seed=seed, device=dev))
cfg = PassConfig(seed=seed, spp=spp)
sess = GuidingSession(w, h, cfg, device=dev)
for f in range(F - 1):
    g, v = frames[f]
    sess.step(GBufferPlanes.from_ref(g, device=dev), VplPlanes.from_ref(v, device=dev), f)
gin = sess.gamma.to_aos().cpu().numpy()
(gp, _), (gc, vc) = frames[F - 2], frames[F - 1]
r = run_pass(cfg, F - 1, GBufferPlanes.from_ref(gc, device=dev), GammaPlanes.from_aos(gin, dev),
             prev=GBufferPlanes.from_ref(gp, device=dev), vpl=VplPlanes.from_ref(vc, device=dev), want_reproj=True)
rep_gpu = r.gamma_reproj.to_aos().cpu().numpy()
gpn, gcn, vcn = _ns(gp), _ns(gc), _ns(vc)
rep = O.reproject(gin, gpn, gcn)
print("gin   ", gin[Y, X])
print("rep o ", rep[Y, X])
print("rep g ", rep_gpu[Y, X])
print("rel   ", np.abs(rep_gpu[Y, X] - rep[Y, X]) / np.maximum(np.abs(rep[Y, X]), 1e-7))
tx = int(np.rint(X + gcn.motion[Y, X, 0]))
ty = int(np.rint(Y + gcn.motion[Y, X, 1]))
print("src", ty, tx, "n_prev", gpn.normal[ty, tx], "n_cur", gcn.normal[Y, X])
relall = np.abs(rep_gpu - rep) / np.maximum(np.abs(rep), 1e-7)
print("whole-frame reproj rel: max", relall.max(), "p99.99", np.percentile(relall, 99.99),
      "n>1e-5", int((relall > 1e-5).sum()), "n>1e-4", int((relall > 1e-4).sum()))
idx = np.argwhere(relall.max(-1) > 1e-5)[:10]
for yy, xx in idx:
    print(yy, xx, relall[yy, xx].max(), rep[yy, xx, :2], rep_gpu[yy, xx, :2])
# dump the pixel for offline analysis
smp = _samples(r, w * h, spp)
p = Y * w + X
np.savez("gpurun_out/pixel_%d_%d.npz" % (Y, X), rep=rep[Y, X], normal=gcn.normal[Y, X], view=gcn.view[Y, X],
         kind=gcn.kind[Y, X], rough=gcn.roughness[Y, X], valid=gcn.valid[Y, X],
         wi_gpu=smp["wi"][p], pdf_gpu=smp["pdf"][p], strat_gpu=smp["strategy"][p], pix=p, seed=seed, frame=F - 1, spp=spp)
