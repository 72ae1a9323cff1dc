"""CPU: host-side pieces of the CLI and metrics (argument/config handling,
PFM/PPM IO), mirroring pg/cli.py:277-338 and pg/metrics.py:50-100."""

import json

import numpy as np
import pytest

from paper_2112_09728_b200 import cli, metrics


def test_pfm_roundtrip_bitwise(tmp_path):
    r = np.random.default_rng(1)
    img = r.standard_normal((7, 9, 3)).astype(np.float32)
    img[0, 0] = [np.inf, -0.0, 1e-40]
    p = str(tmp_path / "a.pfm")
    metrics.write_pfm(img, p)
    back = metrics.read_pfm(p)
    assert back.dtype == np.float32 and back.shape == img.shape
    assert np.array_equal(back.view(np.uint32), img.view(np.uint32))
    raw = open(p, "rb").read()
    assert raw.startswith(b"PF\n9 7\n-1.0\n") and len(raw) == len(b"PF\n9 7\n-1.0\n") + 7 * 9 * 12
    # rows stored bottom-to-top
    first = np.frombuffer(raw[len(b"PF\n9 7\n-1.0\n"):][:9 * 12], "<f4").reshape(9, 3)
    assert np.array_equal(first, img[-1])
    with pytest.raises(ValueError):
        metrics.write_pfm(np.zeros((2, 2)), p)


def test_pfm_errors(tmp_path):
    p = tmp_path / "bad.pfm"
    p.write_bytes(b"P6\n1 1\n-1.0\n")
    with pytest.raises(ValueError, match="not a color PFM"):
        metrics.read_pfm(str(p))
    p.write_bytes(b"PF\n2 2\n-1.0\n" + b"\0" * 10)
    with pytest.raises(ValueError, match="truncated"):
        metrics.read_pfm(str(p))


def test_ppm_tonemap(tmp_path):
    img = np.array([[[0.0, 0.5, 2.0], [1.0, 0.25, -1.0]]], np.float32)
    p = tmp_path / "a.ppm"
    metrics.write_ppm_tonemapped(img, str(p))
    raw = p.read_bytes()
    assert raw.startswith(b"P6\n2 1\n255\n")
    px = np.frombuffer(raw[len(b"P6\n2 1\n255\n"):], np.uint8)
    exp = np.floor(np.clip(img.astype(np.float64), 0, 1) ** (1 / 2.2) * 255 + 0.5).astype(np.uint8).ravel()
    assert np.array_equal(px, exp)
    with pytest.raises(ValueError):
        metrics.write_ppm_tonemapped(img, str(p), exposure=0)


def test_config_precedence(tmp_path):
    c = tmp_path / "cfg.json"
    c.write_text(json.dumps({"width": 20, "spp": 3, "mode": "pg"}))
    args = cli.build_parser().parse_args(["render", "--config", str(c), "--spp", "5"])
    cfg = cli._config_from_args(args)
    assert (cfg.width, cfg.height, cfg.spp, cfg.mode) == (20, 64, 5, "pg")
    c.write_text(json.dumps({"bogus": 1}))
    with pytest.raises(cli.UsageError, match="unknown keys"):
        cli._config_from_args(cli.build_parser().parse_args(["render", "--config", str(c)]))


def test_usage_errors_exit_2(tmp_path):
    assert cli.main(["render", "--frames", "0", "--out", str(tmp_path)]) == 2
    assert cli.main(["render", "--scene", "nope", "--out", str(tmp_path)]) == 2
    assert cli.main(["flicker", "--frames", "1", "--out", str(tmp_path)]) == 2
    with pytest.raises(SystemExit):
        cli.main(["render", "--mode", "xx"])


def test_validate():
    with pytest.raises(cli.UsageError):
        cli.RunConfig(kmax=0).validate()
    with pytest.raises(ValueError):
        cli.RunConfig(max_depth=1).path_config(True)
