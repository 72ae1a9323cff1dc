"""Load the committed golden fixtures (tests/golden/*.npz, produced by the
reference itself through tests/golden/make_golden.py)."""

import os
from types import SimpleNamespace

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
GB_FIELDS = ("valid", "pos", "normal", "depth", "mat", "kind", "albedo", "roughness", "front", "view",
             "motion", "has_history")


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name)))


def gbuf(z, prefix):
    """Reference-style G-buffer namespace, float fields upcast to f64 (the
    exact values the reference was fed)."""
    d = {}
    for k in GB_FIELDS:
        a = z[f"{prefix}gb_{k}"]
        d[k] = a.astype(np.float64) if a.dtype == np.float32 else a
    d["cam_origin"] = z[f"{prefix}gb_cam_origin"]
    h, w = d["valid"].shape
    d["height"], d["width"] = h, w
    return SimpleNamespace(**d)


def gbuf_raw(z, prefix):
    """Same fields at their stored (float32) precision, as dict (device input)."""
    d = {k: z[f"{prefix}gb_{k}"] for k in GB_FIELDS}
    d["cam_origin"] = tuple(float(x) for x in z[f"{prefix}gb_cam_origin"])
    d["height"], d["width"] = d["valid"].shape
    return d


def vpl(z, prefix):
    return SimpleNamespace(valid=z[f"{prefix}vpl_valid"], y=z[f"{prefix}vpl_y"].astype(np.float64),
                           radiance=z[f"{prefix}vpl_radiance"].astype(np.float64),
                           strategy=z[f"{prefix}vpl_strategy"])


def vpl_raw(z, prefix):
    return {k: z[f"{prefix}vpl_{k}"] for k in ("valid", "y", "radiance", "strategy")}


def ulp_diff_f32(a, b):
    """Distance in float32 ulps between two float32 arrays (same sign assumed)."""
    ai = np.asarray(a, np.float32).view(np.int32).astype(np.int64)
    bi = np.asarray(b, np.float32).view(np.int32).astype(np.int64)
    return np.abs(ai - bi)


def rel_err(a, b, floor=1e-7):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.abs(a - b) / np.maximum(np.abs(b), floor)
