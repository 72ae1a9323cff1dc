"""Timing of the device-resident pg frame loop: per
stage CUDA-event times of G-buffer + motion, reproject + depth-0 sampling,
path lanes (NEE, max_depth 4), EM training, at a given resolution / spp, plus
the CPU oracle render on a small sample for the baseline.

    python tools/bench_render.py --scene cornell-occluder --width 1920 --height 1080 --spp 1
"""

import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scene", default="cornell-occluder")
    ap.add_argument("--width", type=int, default=1920)
    ap.add_argument("--height", type=int, default=1080)
    ap.add_argument("--spp", type=int, default=1)
    ap.add_argument("--frames", type=int, default=24)
    ap.add_argument("--warmup", type=int, default=6)
    ap.add_argument("--cpu-sample", type=int, default=96, help="square side of the CPU oracle sample (0: skip)")
    a = ap.parse_args()
    from paper_2112_09728_b200 import cli
    from paper_2112_09728_b200 import scene as S
    from paper_2112_09728_b200.render import gbuffer_planes, render_planes
    from paper_2112_09728_b200.session import run_pass
    scene = S.load_scene(a.scene)
    doc = S.BUILTIN_SCENES[a.scene]()
    k0 = dict(doc["camera"][0])
    k1 = dict(k0, frame=1000, origin=[k0["origin"][0] + 0.3, k0["origin"][1], k0["origin"][2]])
    doc["camera"] = [k0, k1]
    scene = S.scene_from_dict(doc)  # slowly panning camera: reprojection does real work
    cfg = cli.RunConfig(width=a.width, height=a.height, spp=a.spp, mode="pg")
    sess = cli.RenderSession(scene, cfg)
    stages = {k: [] for k in ("gbuffer", "reproject_sample", "render", "train", "frame")}

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    # instrumented copy of RenderSession.run_frame (same calls, events between them)
    for f in range(a.warmup + a.frames):
        cam = S.camera_at(scene, f)
        e0 = ev()
        fgb = gbuffer_planes(sess.dscene, cam, a.width, a.height,
                             prev_cam=sess.prev_cam if sess.gbuf_prev is not None else None,
                             out=sess._gbufs[sess._cur])
        sess._gbufs[sess._cur] = fgb
        e1 = ev()
        pc = sess.pass_config(a.spp)
        if sess.gbuf_prev is not None:
            r = run_pass(pc, f, fgb.planes, sess.gamma, prev=sess.gbuf_prev.planes, want_reproj=True,
                         want_samples=True, out_reproj=sess._spare[0])
            g_rep = r.gamma_reproj
        else:
            r = run_pass(pc, f, fgb.planes, sess.gamma, want_samples=True)
            g_rep = sess.gamma
        e2 = ev()
        rp = render_planes(sess.dscene, fgb, f, cfg.seed, spp=a.spp, max_depth=cfg.max_depth, depth0=r.samples)
        e3 = ev()
        b = run_pass(pc, f, fgb.planes, g_rep, vpl=rp.vpl, want_samples=False, out_gamma=sess._spare[1])
        e4 = ev()
        old = sess.gamma
        sess.gamma = b.gamma
        sess._spare = [g_rep if g_rep is not old else sess._spare[0], old]
        sess.gbuf_prev, sess.prev_cam, sess._cur = fgb, cam, 1 - sess._cur
        torch.cuda.synchronize()
        if f >= a.warmup:
            for k, (x, y) in zip(stages, [(e0, e1), (e1, e2), (e2, e3), (e3, e4), (e0, e4)]):
                stages[k].append(x.elapsed_time(y))
    px = a.width * a.height
    ms = {k: sum(v) / len(v) for k, v in stages.items()}
    seg = float(rp.counters[0].item())
    out = {"metric": "pg_frame_throughput", "value": px / (ms["frame"] * 1e-3) / 1e6, "unit": "Mpix/s",
           "ms_per_frame": ms["frame"], "stages_ms": {k: ms[k] for k in stages if k != "frame"},
           "render_mpix_s": px / (ms["render"] * 1e-3) / 1e6,
           "rays_per_s_render": (seg + px * a.spp * 3) / (ms["render"] * 1e-3),  # scatter + NEE shadow (upper) rays
           "config": {"scene": a.scene, "width": a.width, "height": a.height, "spp": a.spp, "max_depth": 4,
                      "frames": a.frames, "warmup": a.warmup}}
    # image-error kernel (metrics.rel_mse): HBM-bound reduction over two float32 images
    from paper_2112_09728_b200 import _lib
    img = rp.image
    ref = img.flip(0).contiguous()
    n = img.numel()
    scratch = torch.empty(_lib.IMAGE_ERROR_SCRATCH, dtype=torch.float64, device=img.device)
    res = torch.empty(1, dtype=torch.float64, device=img.device)
    big = torch.empty(64 << 20, dtype=torch.float32, device=img.device)  # 256 MB L2 flush
    times = []
    for it in range(12):
        big.fill_(it)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(_lib.lib().pgg_image_error(n, _lib.ptr(img), _lib.ptr(ref), 1, _lib.ptr(scratch), _lib.ptr(res),
                                              _lib.stream_ptr()))
        e1.record()
        torch.cuda.synchronize()
        if it >= 2:
            times.append(e0.elapsed_time(e1))
    t = sorted(times)[len(times) // 2]
    out["image_error"] = {"ms": t, "GB/s": 8.0 * n / (t * 1e-3) / 1e9, "bytes": 8 * n}
    if a.cpu_sample:
        from types import SimpleNamespace

        from oracle import pgg_render_oracle as RO
        n = a.cpu_sample
        cam = S.camera_at(scene, 0)
        t0 = time.perf_counter()
        g = RO.gbuffer(scene, cam, n, n)
        RO.render(scene, 0, 0, SimpleNamespace(**vars(g)), spp=a.spp)
        dt = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": n * n / dt / 1e6, "unit": "Mpix/s", "cores": 1, "kind": "port",
                               "sample": f"oracle gbuffer + pt render, {n}x{n} spp {a.spp}"}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
