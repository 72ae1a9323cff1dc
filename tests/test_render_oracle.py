"""CPU: the render oracle (oracle/pgg_render_oracle.py) reproduces the
reference's own render outputs (tests/golden/render_*.npz), and the scene
loader enforces the reference's validation rules (pg/scene.py:418-573)."""

import json
from types import SimpleNamespace

import numpy as np
import pytest

import golden_io as gio
from oracle import pgg_render_oracle as RO
from paper_2112_09728_b200 import scene as S

CASES = ["cornell_anim", "glossy_box", "corridor"]
GB_FLOAT = ("pos", "normal", "depth", "albedo", "roughness", "view", "motion")


@pytest.mark.parametrize("case", CASES)
def test_oracle_gbuffer_and_render_match_reference(case):
    z = gio.load(f"render_{case}.npz")
    sc = S.scene_from_dict(json.loads(str(z["scene_json"])))
    w, h, fr, spp, seed = (int(z[k]) for k in ("w", "h", "frame", "spp", "seed"))
    gb = RO.gbuffer(sc, S.camera_at(sc, fr), w, h)
    if fr > 0:
        gb.motion, gb.has_history = RO.motion(S.camera_at(sc, fr - 1), gb)
    for k in GB_FLOAT + ("valid", "mat", "kind", "front", "has_history"):
        np.testing.assert_array_equal(getattr(gb, k), z["gb_" + k], err_msg=k)
    g = SimpleNamespace(**vars(gb))
    for k in GB_FLOAT:
        setattr(g, k, getattr(gb, k).astype(np.float32).astype(np.float64))
    for mode in ("pt", "pg"):
        r = RO.render(sc, fr, seed, g, spp=spp, stats=z["pg_stats"] if mode == "pg" else None, want_moments=True)
        for k in ("image", "vpl_valid", "vpl_strategy"):
            np.testing.assert_array_equal(r[k], z[f"{mode}_{k}"], err_msg=(mode, k))
        for k in ("vpl_y", "vpl_radiance", "lum_mean", "lum_var"):
            np.testing.assert_allclose(r[k], z[f"{mode}_{k}"], rtol=1e-13, atol=1e-15, err_msg=(mode, k))
        assert r["mean_path_length"] == float(z[f"{mode}_mean_path_length"])
        assert r["nonfinite"] == int(z[f"{mode}_nonfinite"])


def test_builtin_scenes_load():
    for name in S.BUILTIN_SCENES:
        sc = S.load_scene(name)
        assert sc.num_emitters >= 1
        table, (nm, ns, nq, ne) = sc.pack()
        assert table.shape == (nm * S.MAT_STRIDE + ns * S.SPH_STRIDE + nq * S.QUAD_STRIDE + ne,)
        assert S.camera_is_static(sc)


def _doc(**over):
    d = S.BUILTIN_SCENES["glossy-box"]()
    d.update(over)
    return d


@pytest.mark.parametrize("mutate,msg", [
    (lambda d: d.update(extra=1), "unknown fields"),
    (lambda d: d["materials"][0].update(albedo=[1.5, 0, 0]), "albedo outside"),
    (lambda d: d["materials"][0].update(kind="metal"), "kind must be"),
    (lambda d: d["materials"][1].update(name="white"), "duplicate material"),
    (lambda d: d["primitives"].append({"type": "cone"}), "type must be"),
    (lambda d: d["primitives"].append({"type": "sphere", "center": [0, 0, 0], "radius": 1, "material": "lamp"}),
     "emissive spheres"),
    (lambda d: d["primitives"].append({"type": "quad", "corner": [0, 0, 0], "edge_u": [1, 0, 0],
                                       "edge_v": [2, 0, 0], "material": "white"}), "degenerate quad"),
    (lambda d: d["camera"][0].update(fov_deg=180), "fov_deg"),
    (lambda d: d["camera"][0].update(up=[0, -0.1, 1.88]), "parallel"),
    (lambda d: d.update(materials=[]), "missing or empty"),
])
def test_scene_validation_errors(mutate, msg):
    d = _doc()
    mutate(d)
    with pytest.raises(S.SceneError, match=msg):
        S.scene_from_dict(d)


def test_scene_json_parse_error():
    with pytest.raises(S.SceneError, match="parse error"):
        S.load_scene("{not json")


def test_no_light_rejected():
    d = _doc()
    d["materials"][-1]["emission"] = [0, 0, 0]
    with pytest.raises(S.SceneError, match="no emitters"):
        S.scene_from_dict(d)


def test_camera_interpolation():
    d = _doc()
    k0 = dict(d["camera"][0])
    d["camera"] = [dict(k0, frame=10, origin=[1.5, 1.0, 0.12]), k0]
    sc = S.scene_from_dict(d)
    assert [k.frame for k in sc.keyframes] == [0, 10]
    c5 = S.camera_at(sc, 5)
    np.testing.assert_allclose(c5.origin, [1.25, 1.0, 0.12])
    assert not S.camera_is_static(sc)
    np.testing.assert_allclose(S.camera_at(sc, 50).origin, [1.5, 1.0, 0.12])
