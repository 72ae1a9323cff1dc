"""Training records of single pixels of the 4K 4 spp sequence frame (the
tools/full_frame_parity.py worst Gamma pixels): GPU gather_training_batch
vs the oracle's records, per slot.  Usage: python tools/record_diag.py Y X [Y X ...]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from oracle import pgg_oracle as O  # noqa: E402
from paper_2112_09728_b200 import guide_buffers as GB  # noqa: E402
from paper_2112_09728_b200 import synth  # noqa: E402
from paper_2112_09728_b200.layout import GBufferPlanes, PassConfig, VplPlanes  # noqa: E402
from paper_2112_09728_b200.session import GuidingSession  # noqa: E402
from test_gpu_pass import _ns  # noqa: E402

np.set_printoptions(precision=9, linewidth=180)
dev = torch.device("cuda:0")
import os
w, h, seed, spp, F = (int(v) for v in os.environ.get("RD_CFG", "3840,2160,0,4,5").split(","))
frames = list(synth.sequence(w, h, F, seed=seed, device=dev))
sess = GuidingSession(w, h, PassConfig(seed=seed, spp=spp), device=dev)
for f in range(F - 1):
    g, v = frames[f]
    sess.step(GBufferPlanes.from_ref(g, device=dev), VplPlanes.from_ref(v, device=dev), f)
gin = sess.gamma.to_aos().cpu().numpy()
(gp, _), (gc, vc) = frames[F - 2], frames[F - 1]
gpn, gcn, vcn = _ns(gp), _ns(gc), _ns(vc)
rep = O.reproject(gin, gpn, gcn)
gcn.height, gcn.width = h, w
vcn.height, vcn.width = h, w
args = [int(a) for a in sys.argv[1:]]
for Y, X in zip(args[0::2], args[1::2]):
    p = Y * w + X
    st_g = O.seed_lanes(seed, F - 1, np.arange(h * w), 1)
    recs = GB.gather_training_batch((X, Y), vcn, gcn, GB.GuidingBuffer(w, h, rep), 64, st_g)
    rows = (Y, Y + 1)
    _, parts = O.train(rep, vcn, gcn, 64, seed, F - 1, 10.0, return_parts=True, rows=rows)
    q = X
    slots = np.nonzero(parts.ok[q])[0]
    print(f"pixel ({Y},{X}) records gpu {len(recs)} oracle {len(slots)} stats {rep[Y, X]}")
    for rec, s in zip(recs, slots):
        e = np.abs(rec.sq - parts.sq[q, s]).max()
        flag = " <--" if e > 1e-5 else ""
        cand = int(parts.cand[q, s])
        print(f" slot {s:2d} cand ({cand // w},{cand % w}) sq gpu {rec.sq} ref {parts.sq[q, s]} err {e:.2e} "
              f"w {rec.weight:.6g}/{parts.w[q, s]:.6g} r {parts.r[q, s]:.4g}{flag}")
        if flag:
            d = rec.direction
            print("   dir gpu", d, "normal", gcn.normal[Y, X], "vpl y", vcn.y.reshape(-1, 3)[cand], "pos", gcn.pos[Y, X])
