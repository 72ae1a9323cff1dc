"""Closed-loop drift of the drop-in against the real reference, by patch set:
the reference RenderSession (pgtrace, baseline/_ref) run for 4 guided frames
with (a) all four INTEGRATION.md patches, (b) only the depth-0 sampler, (c)
only reproject + training_pass + lobe_from_stats, (d) no patch but the
reference's depth-0 directions rounded to float32 -- each compared with the
unpatched run (fraction of Gamma channels within 1e-4 relative, max).
usage: [PGG_LIB=...] python tools/integration_diag.py"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
sys.path.append("baseline/_ref")
import golden_io as gio  # noqa: E402
from pgtrace import cli, guide_buffers as pg_gb, mixture as pg_mix, ptrace as pg_pt, scene as sc  # noqa: E402

from paper_2112_09728_b200 import guide_buffers as gb, mixture as mix, ptrace as pt  # noqa: E402


def run(frames=4, w=64, h=48):
    doc = sc.BUILTIN_SCENES["cornell-occluder"]()
    k0 = dict(doc["camera"][0])
    doc["camera"] = [k0, dict(k0, frame=40, origin=[k0["origin"][0] + 0.6, k0["origin"][1] - 0.2, k0["origin"][2]])]
    cfg = cli.RunConfig(scene="cornell-occluder", width=w, height=h, spp=1, mode="pg", frames=frames, seed=3)
    s = cli.RenderSession(sc.scene_from_dict(doc), cfg)
    for f in range(frames):
        s.run_frame(f)
    return np.array(s.gamma.stats, dtype=np.float32)


orig = dict(reproject=pg_gb.reproject, training_pass=pg_gb.training_pass, lobe=pg_mix.lobe_from_stats,
            sfb=pg_pt._sample_first_bounce)


def setp(rep=None, tr=None, lobe=None, sfb=None):
    pg_gb.reproject = rep or orig["reproject"]
    pg_gb.training_pass = tr or orig["training_pass"]
    pg_mix.lobe_from_stats = lobe or orig["lobe"]
    pg_pt._sample_first_bounce = sfb or orig["sfb"]


def f32_dirs(*a, **k):
    wi, pdf, s, v = orig["sfb"](*a, **k)
    return wi.astype(np.float32).astype(np.float64), pdf, s, v


ref = run()
out = {"lib": os.environ.get("PGG_LIB", "default")}
for name, kw in (("all_patched", dict(rep=gb.reproject, tr=gb.training_pass, lobe=mix.lobe_from_stats,
                                      sfb=pt._sample_first_bounce)),
                 ("sampler_only", dict(sfb=pt._sample_first_bounce)),
                 ("em_reproject_lobe_only", dict(rep=gb.reproject, tr=gb.training_pass, lobe=mix.lobe_from_stats)),
                 ("lobe_only", dict(lobe=mix.lobe_from_stats)),
                 ("training_only", dict(tr=gb.training_pass)),
                 ("reproject_only", dict(rep=gb.reproject)),
                 ("ref_f32_directions", dict(sfb=f32_dirs))):
    setp(**kw)
    g = run()
    setp()
    r = gio.rel_err(g, ref)
    out[name] = {"frac_within_1e4": float(np.mean(r <= 1e-4)), "max": float(r.max()),
                 "per_channel_frac": [round(float(np.mean(r[..., c] <= 1e-4)), 5) for c in range(8)],
                 "k_equal": bool(np.array_equal(g[..., 7], ref[..., 7]))}
print(json.dumps(out))

# single-step parity of training_pass on the reference session's own inputs
steps = []


def both(gamma, vpl, gbuf, **kw):
    a = orig["training_pass"](gamma, vpl, gbuf, **kw)
    b = gb.training_pass(gamma, vpl, gbuf, **kw)
    r = gio.rel_err(np.asarray(b.stats), np.asarray(a.stats))
    worst = np.unravel_index(np.argmax(r), r.shape)
    steps.append({"p9999": float(np.percentile(r, 99.99)), "max": float(r.max()),
                  "frac_within_1e4": float(np.mean(r <= 1e-4)), "k_equal": bool(np.array_equal(a.stats[..., 7],
                                                                                                 b.stats[..., 7])),
                  "worst": [int(x) for x in worst], "worst_ref": float(np.asarray(a.stats)[worst]),
                  "worst_got": float(np.asarray(b.stats)[worst]), "worst_in": float(np.asarray(gamma.stats)[worst])})
    return a


pg_gb.training_pass = both
run()
pg_gb.training_pass = orig["training_pass"]
print(json.dumps({"training_single_step": steps}))
