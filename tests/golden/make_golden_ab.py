"""Golden outputs of the reference's `ab` experiment (pg/cli.py:240-272),
made by running the REFERENCE itself in the build container:

    python tests/golden/make_golden_ab.py

Small configuration (32x32, warm-up 24, 8 pairs, 256-spp reference) so the
CPU run takes seconds; tests/test_gpu_cli.py compares the GPU CLI's run_ab
on the same configuration.  Also the flicker series of a guided static-camera run.  Output: tests/golden/ab_small.json
"""

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from pgtrace import cli, metrics  # noqa: E402
from pgtrace import scene as sc  # noqa: E402

CFG = dict(width=32, height=32, warmup=24, pairs=8, ref_spp=256, seed=3)


def main():
    os.environ["PG_THREADS"] = "4"
    out = {"config": CFG}
    for name in ("cornell-occluder", "indirect-corridor", "glossy-box"):
        r = cli.run_ab(sc.load_scene(name), cli.RunConfig(**CFG))
        out[name] = {k: float(r[k]) for k in ("pg_mean_relmse", "pt_mean_relmse", "pg_over_pt")}
        print(name, out[name])
    # SPEC criterion 7 setup (no warm-up): the reference's own ratio
    ucfg = dict(width=64, height=64, warmup=0, pairs=16, ref_spp=1024, seed=4)
    r = cli.run_ab(sc.load_scene("cornell-occluder"), cli.RunConfig(**ucfg))
    out["untrained"] = {"config": ucfg, **{k: float(r[k]) for k in ("pg_mean_relmse", "pt_mean_relmse", "pg_over_pt")}}
    print("untrained", out["untrained"])
    # flicker (pg/cli.py:208-233): static camera, guided warm-up, temporal MSE rows
    fcfg = dict(width=32, height=32, frames=4, warmup=8, mode="pg", seed=5)
    session = cli.RenderSession(sc.load_scene("cornell-occluder"), cli.RunConfig(**fcfg))
    frames = [session.run_frame(f).image for f in range(fcfg["warmup"] + fcfg["frames"])][fcfg["warmup"]:]
    out["flicker"] = {"config": fcfg, "temporal_mse": [r.value for r in metrics.flicker_series(frames)]}
    print("flicker", out["flicker"])
    with open(os.path.join(HERE, "ab_small.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
