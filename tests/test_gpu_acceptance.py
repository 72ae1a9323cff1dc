"""The reference SPEC's acceptance criteria 4, 6, 7 and 8
run end to end on the GPU frame loop (criteria 1-3 and 9:
test_gpu_spec.py; criterion 5: test_gpu_cli.py)."""

import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _scene(name):
    from paper_2112_09728_b200 import scene as S
    return S.load_scene(name)


def test_unbiasedness_ab(cuda_dev):
    """4. cornell-occluder 32x32, PG trained 128 frames, then PG and PT
    accumulate 4096 spp: >= 99 % of pixels agree within 3 combined standard
    errors (per-pixel luminance mean and variance of the lanes)."""
    from paper_2112_09728_b200 import cli
    sc = _scene("cornell-occluder")
    cfg = cli.RunConfig(width=32, height=32, spp=1, seed=2)
    pg = cli.RenderSession(sc, cli.RunConfig(**{**vars(cfg), "mode": "pg"}))
    for f in range(128):
        pg.run_frame(f)
    n = 4096
    a = pg.run_frame(128, spp=n, want_moments=True).to_host()
    b = cli.RenderSession(sc, cfg, mode="pt").run_frame(128, spp=n, want_moments=True).to_host()
    se = np.sqrt(a.lum_var / n + b.lum_var / n)
    agree = np.abs(a.lum_mean - b.lum_mean) <= 3.0 * se + 1e-12
    assert agree.mean() >= 0.99, agree.mean()


def test_flicker_pg_below_pt(cuda_dev):
    """6. Static camera: mean temporal MSE of the guided sequence after the
    warm-up is below plain path tracing's over 64 consecutive frames."""
    from paper_2112_09728_b200 import cli, metrics
    sc = _scene("indirect-corridor")
    base = dict(width=64, height=64, spp=1, seed=1)
    out = {}
    for mode in ("pg", "pt"):
        s = cli.RenderSession(sc, cli.RunConfig(**base, mode=mode))
        if mode == "pg":
            for f in range(128):
                s.run_frame(f)
        frames = [s.run_frame(128 + i).image for i in range(65)]
        out[mode] = np.mean([r.value for r in metrics.flicker_series(frames)])
    assert out["pg"] < out["pt"], out


def test_untrained_equivalence(cuda_dev):
    """7. No warm-up: the guided arm starts from init_stats (pi = 0.05) and
    trains during the pairs.  The SPEC's band [0.9, 1.1] is not met by the
    reference itself on this setup (it already helps: 0.866), so the test
    holds the GPU run to the reference's own ratio
    (tests/golden/ab_small.json['untrained'], made by running pgtrace) and
    checks guiding never hurts."""
    import json

    from paper_2112_09728_b200 import cli
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "ab_small.json")))["untrained"]
    res = cli.run_ab(_scene("cornell-occluder"), cli.RunConfig(**gold["config"]))
    assert res["pg_over_pt"] == pytest.approx(gold["pg_over_pt"], rel=1e-3)
    assert res["pg_over_pt"] <= 1.1


def test_render_determinism(cuda_dev, tmp_path):
    """8. Two runs of the render command with one config give bitwise equal PFMs."""
    from paper_2112_09728_b200 import cli
    outs = []
    for k in range(2):
        d = str(tmp_path / f"r{k}")
        assert cli.main(["render", "--scene", "glossy-box", "--mode", "pg", "--frames", "3", "--width", "48",
                         "--height", "40", "--spp", "2", "--out", d]) == 0
        outs.append([open(os.path.join(d, f"frame_{f:04d}.pfm"), "rb").read() for f in range(3)])
    assert outs[0] == outs[1]
    assert torch.cuda.is_available()
