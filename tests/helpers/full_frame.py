"""Whole-frame parity of the fused pass against the CPU oracle (test
infrastructure: tests/test_gpu_pass.py and tools/full_frame_parity.py).

`run(w, h, spp, F)`: the bench sequence's frame F - 1 with Gamma from F - 1
GPU frames fed to both sides; the GPU pass over the whole frame, the oracle
(oracle/pgg_oracle.py guiding_frame, row chunks in a fork pool -- the
children run numpy only) over every row; returns the error record (Gamma,
k, strategy / validity, directions, pdfs, worst entries)."""
import json
import multiprocessing as mp
import os
import sys
import time
import warnings

import numpy as np
import torch

_here = os.path.dirname(os.path.abspath(__file__))
for _p in (os.path.dirname(os.path.dirname(_here)), os.path.dirname(_here)):
    if _p not in sys.path:
        sys.path.insert(0, _p)
from oracle import pgg_oracle as O  # noqa: E402
from paper_2112_09728_b200 import synth  # noqa: E402
from paper_2112_09728_b200.layout import GammaPlanes, GBufferPlanes, PassConfig, VplPlanes  # noqa: E402
from paper_2112_09728_b200.session import GuidingSession, run_pass  # noqa: E402

G = {}


def _ns(d):
    from types import SimpleNamespace
    return SimpleNamespace(**{k: (v.cpu().numpy().astype(np.float64) if torch.is_tensor(v) and v.dtype == torch.float32
                                  else (v.cpu().numpy() if torch.is_tensor(v) else v)) for k, v in d.items()})


def _samples(res, n, spp):
    d = res.samples.dir.cpu().numpy().reshape(n, spp, 4)
    t = res.samples.tag.cpu().numpy().reshape(n, spp)
    return dict(wi=d[..., :3].astype(np.float64), pdf=d[..., 3].astype(np.float64), strategy=t & 1,
                valid=((t >> 1) & 1).astype(bool))


def rel(a, b):
    return (np.abs(a.astype(np.float64) - b) / np.maximum(np.abs(b.astype(np.float64)), 1e-7)).astype(np.float32)


def work(rows):
    r0, r1 = rows
    g = G
    w, spp = g["w"], g["spp"]
    _, osmp, otr = O.guiding_frame(g["gin"], g["gpn"], g["gcn"], g["vcn"], g["seed"], g["frame"], spp=spp,
                                   kmax=g["kmax"], radius=g["radius"], nee_draws=g.get("nee", 3), rows=(r0, r1))
    band = slice(r0 * w, r1 * w)
    gam = g["got"][r0:r1]
    sm = {k: v[band] for k, v in g["smp"].items()}
    direrr = np.abs(sm["wi"] - osmp["wi"]).max(-1).astype(np.float32)
    both = sm["valid"] & osmp["valid"]
    prel = np.where(both, rel(sm["pdf"], osmp["pdf"]), 0).astype(np.float32)
    out = dict(gam_rel=rel(gam, otr), k_bad=int(np.count_nonzero(gam[..., 7] != otr[..., 7])),
               strat_bad=int(np.count_nonzero(sm["strategy"] != osmp["strategy"])),
               valid_bad=int(np.count_nonzero(sm["valid"] != osmp["valid"])),
               dir_err=direrr, pdf_rel=prel, worst=[])
    gr = out["gam_rel"]
    out["worst_gamma"] = []
    for i in np.argsort(gr.ravel())[::-1][:3]:
        yy, xx, c = np.unravel_index(int(i), gr.shape)
        out["worst_gamma"].append(dict(y=r0 + int(yy), x=int(xx), ch=int(c), rel=float(gr[yy, xx, c]),
                                       got=float(gam[yy, xx, c]), ref=float(otr[yy, xx, c]),
                                       gin=g["gin"][r0 + yy, xx].tolist(), got_px=gam[yy, xx].tolist(),
                                       ref_px=otr[yy, xx].tolist()))
    out["worst_pdf"] = []
    for i in np.argsort(prel.ravel())[::-1][:3]:
        pp, ss = divmod(int(i), spp)
        yy, xx = r0 + pp // w, pp % w
        out["worst_pdf"].append(dict(y=yy, x=xx, lane=ss, rel=float(prel.ravel()[i]), pdf=float(sm["pdf"][pp, ss]),
                                     ref=float(osmp["pdf"][pp, ss]), strategy=int(osmp["strategy"][pp, ss]),
                                     kind=int(g["gcn"].kind[yy, xx]), rough=float(g["gcn"].roughness[yy, xx]),
                                     ndotv=float(np.dot(g["gcn"].normal[yy, xx], g["gcn"].view[yy, xx])),
                                     wi=osmp["wi"][pp, ss].tolist(), n=g["gcn"].normal[yy, xx].tolist(),
                                     stats=g["gin"][yy, xx].tolist()))
    for i in np.argsort(direrr.ravel())[::-1][:3]:
        p, s = divmod(int(i), spp)
        out["worst"].append(dict(y=r0 + p // w, x=p % w, lane=s, dir_err=float(direrr.ravel()[i]),
                                 strategy=int(osmp["strategy"][p, s])))
    return out


def compare(gin, gpn, gcn, vcn, got, smp, w, h, spp, seed, frame, k_max=64, radius=10.0, chunk=24, procs=None,
            label="", nee_draws=3):
    """GPU outputs (Gamma' AoS `got`, samples dict `smp`) of one pass against
    the oracle's guiding_frame on the same inputs, every row."""
    G.clear()
    G.update(w=w, spp=spp, seed=seed, frame=frame, kmax=k_max, radius=radius, gin=gin, gpn=gpn, gcn=gcn, vcn=vcn,
             got=got, smp=smp, nee=nee_draws)
    t0 = time.time()
    bands = [(a, min(h, a + chunk)) for a in range(0, h, chunk)]
    with warnings.catch_warnings():
        # the children run numpy only (no CUDA, no locks of the parent's threads)
        warnings.filterwarnings("ignore", message=".*use of fork\\(\\) may lead to deadlocks.*")
        with mp.get_context("fork").Pool(procs or os.cpu_count()) as pool:
            res = pool.map(work, bands)
    gam = np.concatenate([x["gam_rel"] for x in res])
    de = np.concatenate([x["dir_err"] for x in res])
    pr = np.concatenate([x["pdf_rel"] for x in res])
    worst = sorted([wl for x in res for wl in x["worst"]], key=lambda d: -d["dir_err"])[:8]
    return dict(config=label or f"{w}x{h} {spp} spp frame {frame}, k_max {k_max}, radius {radius}", pixels=w * h,
                lanes=w * h * spp, oracle_seconds=round(time.time() - t0, 1),
                gamma_rel_p9999=float(np.percentile(gam, 99.99)), gamma_rel_max=float(gam.max()),
                gamma_channels_gt_1e4=int(np.count_nonzero(gam > 1e-4)),
                k_mismatches=sum(x["k_bad"] for x in res), strategy_mismatches=sum(x["strat_bad"] for x in res),
                valid_mismatches=sum(x["valid_bad"] for x in res),
                dir_abs_max=float(de.max()), dir_lanes_gt_1e5=int(np.count_nonzero(de > 1e-5)),
                dir_lanes_gt_3e6=int(np.count_nonzero(de > 3e-6)),
                pdf_rel_p9999=float(np.percentile(pr, 99.99)), pdf_rel_max=float(pr.max()), worst_dirs=worst,
                worst_pdf=sorted([wp for x in res for wp in x["worst_pdf"]], key=lambda d: -d["rel"])[:8],
                worst_gamma=sorted([wg for x in res for wg in x["worst_gamma"]], key=lambda d: -d["rel"])[:8])


def run(w, h, spp, F, seed=0, chunk=24, procs=None, verbose=True, k_max=64, radius=10.0):
    """The bench sequence's frame F - 1 (Gamma from F - 1 GPU frames)."""
    dev = torch.device("cuda:0")
    frames = list(synth.sequence(w, h, F, seed=seed, device=dev))
    cfg = PassConfig(seed=seed, spp=spp, k_max=k_max, neighbor_radius=radius)
    sess = GuidingSession(w, h, cfg, device=dev)
    for f in range(F - 1):
        g, v = frames[f]
        sess.step(GBufferPlanes.from_ref(g, device=dev), VplPlanes.from_ref(v, device=dev), f)
    gin = sess.gamma.to_aos().cpu().numpy()
    (gp, _), (gc, vc) = frames[F - 2], frames[F - 1]
    r = run_pass(cfg, F - 1, GBufferPlanes.from_ref(gc, device=dev), GammaPlanes.from_aos(gin, dev),
                 prev=GBufferPlanes.from_ref(gp, device=dev), vpl=VplPlanes.from_ref(vc, device=dev))
    args = (gin, _ns(gp), _ns(gc), _ns(vc), r.gamma.to_aos().cpu().numpy(), _samples(r, w * h, spp))
    del frames, sess, r
    torch.cuda.empty_cache()
    rec = compare(*args, w, h, spp, seed, F - 1, k_max, radius, chunk, procs)
    if verbose:
        print(json.dumps(rec), flush=True)
    return rec
