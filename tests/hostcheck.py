"""Test-only host build of the device bodies (csrc/pgg_hostcheck.cpp).

Compiles the same pgg_pass.cuh / pgg_math.cuh the CUDA kernels use with g++
into build/libpgg_hostcheck.so and drives it with NumPy buffers in the packed
layout, so the CPU suite can hold the device formulas to the oracle without
a GPU.  Never used by the product package.
"""

import ctypes
import os
import subprocess

import numpy as np

from paper_2112_09728_b200 import _lib

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
CSRC = os.path.join(ROOT, "paper_2112_09728_b200", "csrc")
OUT = os.path.join(ROOT, "build", "libpgg_hostcheck.so")
SRCS = [os.path.join(CSRC, f) for f in ("pgg_hostcheck.cpp", "pgg_pass.cuh", "pgg_math.cuh")] + [
    os.path.join(ROOT, "include", "pgg.h")]

_hc = None


def build():
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    if os.path.exists(OUT) and os.path.getmtime(OUT) >= max(os.path.getmtime(s) for s in SRCS):
        return OUT
    cmd = ["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fPIC", "-shared", "-I/usr/local/cuda/include",
           "-I" + os.path.join(ROOT, "include"), "-I" + CSRC, "-x", "c++", SRCS[0], "-o", OUT + ".tmp"]
    subprocess.run(cmd, check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT


def lib():
    global _hc
    if _hc is None:
        _hc = ctypes.CDLL(build())
        P = ctypes.POINTER
        _hc.pgghc_guiding_pass.argtypes = [P(_lib.Config), P(_lib.GBuffer), P(_lib.GBuffer), P(_lib.GammaIn),
                                           P(_lib.Vpl), P(_lib.GammaOut), P(_lib.GammaOut), P(_lib.Samples),
                                           ctypes.c_void_p]
        for n in ("pgghc_trunc_mass", "pgghc_lobe_f", "pgghc_sq_to_dir", "pgghc_dir_to_sq", "pgghc_box_muller",
                  "pgghc_disk_offset", "pgghc_neighbor_budget"):
            getattr(_hc, n).restype = ctypes.c_int
        _hc.pgghc_disk_offset.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double,
                                          ctypes.c_void_p]
        _hc.pgghc_neighbor_budget.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p]
    return _hc


def P(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


# ---- NumPy packers mirroring k_pack_gbuffer / k_pack_vpl / k_gamma_split

def pack_gbuffer(g):
    f32 = np.float32
    valid = np.asarray(g["valid"]).astype(bool)
    h, w = valid.shape
    flags = (valid.astype(np.uint8) | (np.asarray(g["has_history"]).astype(np.uint8) << 1)
             | ((np.asarray(g["kind"]) == 1).astype(np.uint8) << 2))
    nd = np.concatenate([np.asarray(g["normal"], f32), np.asarray(g["depth"], f32)[..., None]], -1)
    pr = np.concatenate([np.asarray(g["pos"], f32), np.asarray(g["roughness"], f32)[..., None]], -1)
    alb = np.asarray(g["albedo"], f32)
    va = np.concatenate([np.asarray(g["view"], f32), alb[..., :1]], -1)
    am = np.concatenate([alb[..., 1:3], np.asarray(g["motion"], f32)], -1)
    return dict(flags=np.ascontiguousarray(flags), nd=np.ascontiguousarray(nd), pr=np.ascontiguousarray(pr),
                va=np.ascontiguousarray(va), am=np.ascontiguousarray(am), h=h, w=w,
                cam=tuple(float(c) for c in g["cam_origin"]))


def pack_vpl(v):
    f32 = np.float32
    use = (np.asarray(v["valid"]).astype(bool) & (np.asarray(v["strategy"]) == 0)).astype(f32)
    y = np.concatenate([np.asarray(v["y"], f32), use[..., None]], -1)
    L = np.concatenate([np.asarray(v["radiance"], f32), np.zeros(use.shape + (1,), f32)], -1)
    return dict(y=np.ascontiguousarray(y), L=np.ascontiguousarray(L))


def split_gamma(stats):
    s = np.ascontiguousarray(np.asarray(stats, np.float32))
    return np.ascontiguousarray(s[..., :4]), np.ascontiguousarray(s[..., 4:])


def frame_key(seed, frame, stream):
    from oracle import pgg_oracle as O
    return int(O.frame_key(seed, frame, stream))


def run_pass(cur, gamma_in, seed, frame, prev=None, vpl=None, spp=1, nee_draws=3, k_max=64, radius=10.0,
             want_reproj=True, want_samples=True, rotate_mean=True):
    """Drive pgghc_guiding_pass on NumPy inputs; returns dict of outputs."""
    L = lib()
    cg = pack_gbuffer(cur)
    h, w = cg["h"], cg["w"]
    c = _lib.Config()
    c.width, c.height, c.row0, c.rows = w, h, 0, h
    c.spp, c.nee_draws, c.k_max, c.rotate_mean = spp, nee_draws, k_max, 1 if rotate_mean else 0
    c.radius, c.depth_rel_tol, c.normal_dot_min, c.rough_min_guide = radius, 0.1, 0.9, 0.05
    pg = pack_gbuffer(prev) if prev is not None else None
    if pg is not None:
        for i in range(3):
            c.prev_cam[i] = pg["cam"][i]
    c.key_sample = frame_key(seed, frame, 0)
    c.key_train = frame_key(seed, frame, 1)
    gb = _lib.GBuffer(P(cg["flags"]), P(cg["nd"]), P(cg["pr"]), P(cg["va"]), P(cg["am"]), 0, h)
    gbp = _lib.GBuffer(P(pg["flags"]), P(pg["nd"]), P(pg["pr"]), P(pg["va"]), P(pg["am"]), 0, h) if pg else None
    g0, g1 = split_gamma(gamma_in)
    gin = _lib.GammaIn(P(g0), P(g1), 0, h)
    out = {}
    r0 = np.zeros((h, w, 4), np.float32)
    r1 = np.zeros((h, w, 4), np.float32)
    grep = _lib.GammaOut(P(r0), P(r1)) if want_reproj else None
    vp = pack_vpl(vpl) if vpl is not None else None
    vplabi = _lib.Vpl(P(vp["y"]), P(vp["L"]), 0, h) if vp else None
    o0 = np.zeros((h, w, 4), np.float32)
    o1 = np.zeros((h, w, 4), np.float32)
    gout = _lib.GammaOut(P(o0), P(o1)) if vp else None
    sd = np.zeros((h, w, spp, 4), np.float32)
    st = np.zeros((h, w, spp), np.uint8)
    smp = _lib.Samples(P(sd), P(st)) if want_samples else None
    miss = np.zeros(1, np.int32)
    ref = ctypes.byref
    rc = L.pgghc_guiding_pass(ref(c), ref(gb), ref(gbp) if gbp else None, ref(gin), ref(vplabi) if vplabi else None,
                              ref(grep) if grep else None, ref(gout) if gout else None, ref(smp) if smp else None,
                              P(miss))
    assert rc == 0
    if want_reproj:
        out["gamma_reproj"] = np.concatenate([r0, r1], -1)
    if vp:
        out["gamma_trained"] = np.concatenate([o0, o1], -1)
    if want_samples:
        out["wi"] = sd[..., :3].reshape(h * w, spp, 3)
        out["pdf"] = sd[..., 3].reshape(h * w, spp)
        out["strategy"] = (st & 1).reshape(h * w, spp)
        out["valid"] = ((st >> 1) & 1).astype(bool).reshape(h * w, spp)
    out["halo_misses"] = int(miss[0])
    return out
