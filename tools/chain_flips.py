"""Where does the multi-frame GPU trajectory leave the oracle's, and why?

Runs the fused GPU chain and the CPU oracle chain side by side (SURVEY.md
8a trajectory policy) and, every frame, also runs the oracle ONE step from
the GPU's own previous Gamma ("re-anchored"): that separates the kernel's
per-step error (re-anchored vs GPU: the single-kernel policy) from the
amplification of earlier float32 differences by the reference's
discontinuities (chain vs re-anchored).  For every pixel channel outside
1e-4 at the end it reports the first frame where the pixel's discrete state
diverged between the two chains:
  reproj   reprojection accept/reject differs (gate or mean-rotation z < 0)
  reset    the lobe's lambda_min < 1e-6 reset decision differs
  k        k (number of informative EM batches) differs
  none     no discrete divergence: continuous drift only
Usage: python tools/chain_flips.py [W H FRAMES SEED] [--json out.json]"""
import json
import sys
from types import SimpleNamespace

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import pgg_oracle as O  # noqa: E402
from paper_2112_09728_b200 import synth  # noqa: E402
from paper_2112_09728_b200.layout import GammaPlanes, GBufferPlanes, PassConfig, VplPlanes  # noqa: E402
from paper_2112_09728_b200.session import GuidingSession, run_pass  # noqa: E402


def ns(d):
    return SimpleNamespace(**{k: (v.cpu().numpy().astype(np.float64) if torch.is_tensor(v) and v.dtype == torch.float32
                                  else (v.cpu().numpy() if torch.is_tensor(v) else v)) for k, v in d.items()})


def rel(a, b):
    return np.abs(a.astype(np.float64) - b) / np.maximum(np.abs(b.astype(np.float64)), 1e-7)


def accepted(gam_prev, g_rep):
    """reprojection accepted where the reprojected Gamma is not init_stats"""
    fresh = np.array([0.5, 0.5, 0.5, 0.5, 0.25, 0.0, 0.05, 0.0], np.float32)
    return ~np.all(g_rep == fresh, axis=-1)


def main(w=160, h=120, frames=4, seed=9, out=None):
    dev = torch.device("cuda:0")
    cfg = PassConfig(seed=seed, spp=1)
    sess = GuidingSession(w, h, cfg, device=dev)
    gam = O.fresh_stats(h * w).reshape(h, w, 8).astype(np.float32)
    prev = None
    prev_dev = None
    first = {}  # pixel -> (frame, cause)
    report = {"config": dict(w=w, h=h, frames=frames, seed=seed), "frames": []}
    for f, (g, v) in enumerate(synth.sequence(w, h, frames, seed=seed)):
        gpu_in = sess.gamma.to_aos().cpu().numpy()
        cur = GBufferPlanes.from_ref(g, device=dev)
        vp = VplPlanes.from_ref(v, device=dev)
        # the GPU step with its reprojected Gamma exposed
        r = run_pass(cfg, f, cur, sess.gamma, prev=prev_dev, vpl=vp, want_reproj=prev_dev is not None)
        gpu_rep = r.gamma_reproj.to_aos().cpu().numpy() if prev_dev is not None else gpu_in
        sess.step(cur, vp, f)
        gpu = sess.gamma.to_aos().cpu().numpy()
        assert np.array_equal(gpu, r.gamma.to_aos().cpu().numpy())
        gn, vn = ns(g), ns(v)
        o_rep, _, o_tr = O.guiding_frame(gam, prev, gn, vn, seed, f, spp=1)        # oracle chain
        a_rep, _, a_tr = O.guiding_frame(gpu_in, prev, gn, vn, seed, f, spp=1)     # re-anchored on the GPU's input
        valid = gn.valid.astype(bool)
        step = rel(gpu, a_tr)
        chain = rel(gpu, o_tr)
        # discrete divergences between the two chains this frame
        rep_flip = (accepted(None, o_rep) != accepted(None, gpu_rep)) & valid
        lo = O.lobe(o_rep.reshape(-1, 8).astype(np.float64)).reset.reshape(h, w)
        lg = O.lobe(gpu_rep.reshape(-1, 8).astype(np.float64)).reset.reshape(h, w)
        reset_flip = (lo != lg) & valid
        k_flip = (o_tr[..., 7] != gpu[..., 7])
        for cause, m in (("reproj", rep_flip), ("reset", reset_flip), ("k", k_flip)):
            for yy, xx in zip(*np.nonzero(m)):
                first.setdefault((int(yy), int(xx)), (f, cause))
        fr = {"frame": f,
              "step_p9999": float(np.percentile(step, 99.99)), "step_max": float(step.max()),
              "step_k_equal": bool(np.array_equal(gpu[..., 7], a_tr[..., 7])),
              "step_reproj_equal_frac": float(np.mean(rel(gpu_rep, a_rep) <= 1e-4)),
              "chain_frac_1e4": float(np.mean(chain <= 1e-4)), "chain_max": float(chain.max()),
              "chain_k_equal_frac": float(np.mean(gpu[..., 7] == o_tr[..., 7])),
              "reproj_flips": int(rep_flip.sum()), "reset_flips": int(reset_flip.sum()),
              "k_flips": int(k_flip.sum())}
        report["frames"].append(fr)
        print(json.dumps(fr), flush=True)
        gam, prev, prev_dev = o_tr, gn, cur
    bad = np.argwhere(chain > 1e-4)  # (y, x, channel)
    causes = {}
    rows = []
    for yy, xx, c in bad:
        fc = first.get((int(yy), int(xx)), (None, "none"))
        causes[fc[1]] = causes.get(fc[1], 0) + 1
        rows.append([int(yy), int(xx), int(c), float(chain[yy, xx, c]), fc[0], fc[1]])
    report["final"] = {"channels": int(chain.size), "outside_1e4": int(len(bad)),
                       "frac_within_1e4": float(np.mean(chain <= 1e-4)), "by_cause": causes,
                       "pixels_outside": int(len({(r[0], r[1]) for r in rows}))}
    report["outside"] = rows
    # the reference's own conditioning: its chain vs the same chain with Gamma
    # channels 0-5 nudged by one float32 ulp after frame 0 (SURVEY 8a drift.py)
    frames_ns = [(ns(g), ns(v)) for g, v in synth.sequence(w, h, frames, seed=seed)]
    ulp = []
    for pseed in (0, 1):
        a = O.fresh_stats(h * w).reshape(h, w, 8).astype(np.float32)
        b = a.copy()
        pv = None
        rng = np.random.default_rng(pseed)
        for f, (gn, vn) in enumerate(frames_ns):
            _, _, a = O.guiding_frame(a, pv, gn, vn, seed, f, spp=1)
            _, _, b = O.guiding_frame(b, pv, gn, vn, seed, f, spp=1)
            if f == 0:
                sgn = rng.choice([-1.0, 1.0], size=b[..., :6].shape).astype(np.float32)
                b[..., :6] = np.nextafter(b[..., :6], b[..., :6] + sgn)
            pv = gn
        ulp.append(float(np.mean(rel(b, a) <= 1e-4)))
    report["final"]["reference_1ulp_perturbed_frac_within_1e4"] = ulp
    print(json.dumps(report["final"]), flush=True)
    if out:
        with open(out, "w") as fh:
            json.dump(report, fh, indent=1)


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    out = sys.argv[sys.argv.index("--json") + 1] if "--json" in sys.argv else None
    if out in args:
        args.remove(out)
    main(*[int(x) for x in args], out=out)
