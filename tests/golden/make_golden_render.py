"""Golden vectors of the render pass, produced by running the REFERENCE
itself (build container only: needs /root/reference).

    python tests/golden/make_golden_render.py

For each case it stores the reference's G-buffer (gbuffer_pass +
motion_vectors), the image, VPLs, path statistics and luminance moments of
render_frame, in pt mode and in pg mode (Gamma from a few reference
RenderSession frames).  The G-buffer handed to render_frame is the float32
rounding of the reference's own (upcast back to float64), because the
device G-buffer is float32; the unrounded one is stored too for the G-buffer
kernel's own check.

Output: tests/golden/render_<case>.npz
"""

import json
import os
import sys
from dataclasses import replace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from pgtrace import cli, ptrace  # noqa: E402
from pgtrace import scene as sc  # noqa: E402

GB_FLOAT = ("pos", "normal", "depth", "albedo", "roughness", "view", "motion")
GB_ALL = GB_FLOAT + ("valid", "mat", "kind", "front", "has_history")


def animated(name):
    """A built-in scene with a second camera keyframe (moving camera -> motion vectors)."""
    doc = sc.BUILTIN_SCENES[name]()
    k0 = dict(doc["camera"][0])
    k1 = dict(k0, frame=8, origin=[k0["origin"][0] + 0.12, k0["origin"][1] - 0.05, k0["origin"][2] + 0.04],
              look_at=[k0["look_at"][0] + 0.08, k0["look_at"][1], k0["look_at"][2]])
    doc["camera"] = [k0, k1]
    return doc


def rounded(gb):
    g = replace(gb)
    for k in GB_FLOAT:
        setattr(g, k, getattr(gb, k).astype(np.float32).astype(np.float64))
    return g


def case(name, doc, w, h, frame, spp, pg_frames, seed):
    scene = sc.scene_from_dict(doc)
    out = {"scene_json": json.dumps(doc), "scene_name": name, "w": w, "h": h, "frame": frame, "spp": spp, "seed": seed}
    cam = sc.camera_at(scene, frame)
    gb = ptrace.gbuffer_pass(scene, frame, (w, h))
    if frame > 0:
        m, has = ptrace.motion_vectors(sc.camera_at(scene, frame - 1), cam, gb)
        gb.motion, gb.has_history = m, has
    for k in GB_ALL:
        out["gb_" + k] = getattr(gb, k)
    gr = rounded(gb)
    pcfg = ptrace.PathConfig(max_depth=4, spp=spp)
    r = ptrace.render_frame(scene, frame, None, pcfg, seed, gbuf=gr, want_moments=True)
    for k, v in (("image", r.image), ("vpl_valid", r.vpl.valid), ("vpl_y", r.vpl.y),
                 ("vpl_radiance", r.vpl.radiance), ("vpl_strategy", r.vpl.strategy),
                 ("lum_mean", r.lum_mean), ("lum_var", r.lum_var)):
        out["pt_" + k] = v
    out["pt_mean_path_length"] = r.mean_path_length
    out["pt_nonfinite"] = r.nonfinite_count
    # pg: Gamma after `pg_frames` reference frames, then one guided render
    cfg = cli.RunConfig(width=w, height=h, spp=1, mode="pg", seed=seed)
    sess = cli.RenderSession(scene, cfg)
    for f in range(pg_frames):
        sess.run_frame(frame - pg_frames + f if frame >= pg_frames else f)
    stats = sess.gamma.stats_for_render().astype(np.float32)
    out["pg_stats"] = stats
    pcfg = ptrace.PathConfig(max_depth=4, spp=spp, guiding=True)
    r = ptrace.render_frame(scene, frame, stats, pcfg, seed, gbuf=gr, want_moments=True)
    for k, v in (("image", r.image), ("vpl_valid", r.vpl.valid), ("vpl_y", r.vpl.y),
                 ("vpl_radiance", r.vpl.radiance), ("vpl_strategy", r.vpl.strategy),
                 ("lum_mean", r.lum_mean), ("lum_var", r.lum_var)):
        out["pg_" + k] = v
    out["pg_mean_path_length"] = r.mean_path_length
    out["pg_nonfinite"] = r.nonfinite_count
    return out


def main():
    os.environ["PG_THREADS"] = "1"
    cases = [
        ("cornell_anim", animated("cornell-occluder"), 48, 40, 3, 2, 3, 7),
        ("glossy_box", sc.BUILTIN_SCENES["glossy-box"](), 40, 32, 2, 2, 2, 3),
        ("corridor", sc.BUILTIN_SCENES["indirect-corridor"](), 40, 32, 1, 3, 1, 11),
    ]
    for c in cases:
        out = case(*c)
        np.savez_compressed(os.path.join(HERE, f"render_{c[0]}.npz"), **out)
        print(c[0], "ok", out["pt_mean_path_length"], out["pg_mean_path_length"])


if __name__ == "__main__":
    main()
