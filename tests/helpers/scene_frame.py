"""Whole-frame parity of the fused pass on RENDERED inputs (test
infrastructure: tests/test_gpu_pass.py, tools/scene_parity.py).  `one(name)`:
the GPU frame loop (cli.RenderSession) runs F - 1 guided frames of a
built-in scene, then frame F's G-buffer (k_gbuffer), its VPLs (the GPU path
tracer fed by the pass's own depth-0 samples) and the trained Gamma go to
the fused pass and to the oracle's guiding_frame (helpers.full_frame.compare)."""
import json

import numpy as np
import torch

from helpers.full_frame import _samples, compare  # noqa: E402
from paper_2112_09728_b200 import cli, ptrace  # noqa: E402
from paper_2112_09728_b200 import scene as S  # noqa: E402
from paper_2112_09728_b200.render import gbuffer_planes, render_planes  # noqa: E402
from paper_2112_09728_b200.session import run_pass  # noqa: E402


def ns_vpl(vp):
    vy = vp.y.cpu().numpy().astype(np.float64)
    vl = vp.L.cpu().numpy()
    code = vl[..., 3].astype(np.int32)
    from types import SimpleNamespace
    return SimpleNamespace(valid=(code & 1).astype(bool), y=vy[..., :3].copy(), radiance=vl[..., :3].astype(np.float64),
                           strategy=(code >> 1).astype(np.uint8))


def one(name, F=6, w=1920, h=1080, seed=0):
    sc = S.load_scene(name)
    cfg = cli.RunConfig(width=w, height=h, spp=1, mode="pg", seed=seed)
    sess = cli.RenderSession(sc, cfg)
    for f in range(F - 1):
        sess.run_frame(f)
    gin = sess.gamma.to_aos().cpu().numpy()
    prev_fgb, prev_cam = sess.gbuf_prev, sess.prev_cam
    gpn = ptrace.gbuffer_from_planes(prev_fgb, prev_cam.origin)
    f = F - 1
    cam = S.camera_at(sc, f)
    fgb = gbuffer_planes(sess.dscene, cam, w, h, prev_cam=prev_cam)
    pc = sess.pass_config(1)
    a = run_pass(pc, f, fgb.planes, sess.gamma, prev=prev_fgb.planes, want_reproj=True, want_samples=True)
    rp = render_planes(sess.dscene, fgb, f, seed, spp=1, max_depth=cfg.max_depth, depth0=a.samples)
    # the fused pass on frame F's inputs (what the benchmark measures)
    r = run_pass(pc, f, fgb.planes, sess.gamma, prev=prev_fgb.planes, vpl=rp.vpl)
    gcn = ptrace.gbuffer_from_planes(fgb, cam.origin)
    rec = compare(gin, gpn, gcn, ns_vpl(rp.vpl), r.gamma.to_aos().cpu().numpy(), _samples(r, w * h, 1), w, h, 1,
                  seed, f, label=f"{name} {w}x{h} frame {f} (rendered G-buffer / VPLs, Gamma from {f} guided frames)",
                  nee_draws=pc.nee_draws)
    rec["trained_frac"] = float((gin[..., 7] >= 1).mean())
    print(json.dumps({k: v for k, v in rec.items() if not k.startswith("worst")}), flush=True)
    return rec
