"""CPU oracle for the screen-space guiding pass.

TEST INFRASTRUCTURE ONLY.  This module restates, in float64 NumPy, the
algorithm of the reference package ``pgtrace`` (arXiv 2112.09728 desk-scale
reimplementation, mounted read-only at /root/reference/pkg/src/pgtrace, "pg/"
below) for the four parts of the guiding pass: Gamma reprojection, the lobe
(covariance, Cholesky, truncation mass), guided first-bounce sampling with
the one-sample mixture pdf, and the online weighted-EM training pass.

Who may use it: ``tests/`` (as the parity checker), ``__graft_entry__.smoke``
(checker) and ``bench.py`` (the ``cpu_baseline`` leg and ``--impl reference``).
The product package ``paper_2112_09728_b200`` never imports it.

Pinning: the restatement is checked against golden vectors produced by the
reference itself (``tests/golden/make_golden.py`` imports /root/reference in
the build container and commits ``tests/golden/*.npz``) and against the SPEC
known-answer examples.  Where SPEC prose and code
disagree the reference *code* is followed.

Arrays use the reference's own field names so a reader can lay this file
next to pg/guide_buffers.py; the functions are organised per pixel/lane
rather than per reference module.
"""

from types import SimpleNamespace

import numpy as np
from scipy.special import ndtr

# ---------------------------------------------------------------------------
# constants (pg/mixture.py:19-31, pg/guide_buffers.py:18-20, pg/ptrace.py:32)

MEAN_X, MEAN_Y, M2_XX, M2_YY, M2_XY, W_SUM, MIX_PI, EPOCH = range(8)
PI_LO, PI_HI = 0.05, 0.95
RIDGE = 1e-4
EIG_FLOOR = 1e-6
RESET_VAR = 0.05
Z_FLOOR = 1e-4
KMAX = 64
GAUSS_TRIES = 16
STRAT_BRDF, STRAT_GAUSS = 0, 1
DIFFUSE, GLOSSY = 0, 1
RADIUS = 10.0
SLOTS = 20
ROUGH_MIN_GUIDE = 0.05
LUMA = (0.2126, 0.7152, 0.0722)

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
PCG_MUL = np.uint64(6364136223846793005)
PCG_ADD = np.uint64(1442695040888963407)


# ---------------------------------------------------------------------------
# PCG32 lanes (pg/rng.py:15-55)

def splitmix64(x):
    """SplitMix64 finaliser, wrapping uint64 arithmetic (pg/rng.py:15-22)."""
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def frame_key(seed, frame, stream=0):
    """Per-(seed, frame, stream) hash prefix of the key chain (pg/rng.py:34-36).

    Lane-independent, so the device computes it once on the host."""
    h = splitmix64(np.uint64(int(seed) & 0xFFFFFFFFFFFFFFFF))
    h = splitmix64(h ^ splitmix64(np.uint64(frame)))
    with np.errstate(over="ignore"):
        sid = np.uint64(stream) + np.uint64(0xA02BDBF7BB3C0A7)
    return splitmix64(h ^ splitmix64(sid))


def seed_lanes(seed, frame, lanes, stream=0):
    """PCG32 state per lane after the warm-up step (pg/rng.py:25-39)."""
    h = frame_key(seed, frame, stream)
    s = splitmix64(h ^ splitmix64(np.asarray(lanes, dtype=np.uint64)))
    with np.errstate(over="ignore"):
        return s * PCG_MUL + PCG_ADD


def draw_u32(state):
    """XSH-RR output of the current state, then one LCG step, in place
    (pg/rng.py:42-50)."""
    old = state.copy()
    with np.errstate(over="ignore"):
        state *= PCG_MUL
        state += PCG_ADD
    xs = (((old >> np.uint64(18)) ^ old) >> np.uint64(27)).astype(np.uint32)
    rot = (old >> np.uint64(59)).astype(np.uint32)
    return (xs >> rot) | (xs << ((np.uint32(32) - rot) & np.uint32(31)))


def lcg_distance(a, b, limit=64):
    """Number of LCG steps from states a to states b (< limit), per lane."""
    cur = np.array(a, dtype=np.uint64, copy=True)
    n = np.full(cur.shape, -1, dtype=np.int64)
    n[cur == b] = 0
    for i in range(1, limit):
        with np.errstate(over="ignore"):
            cur = cur * PCG_MUL + PCG_ADD
        n[(n < 0) & (cur == b)] = i
    assert np.all(n >= 0), "state not reachable within the limit"
    return n


def draw_unit(state):
    """u32 * 2^-32 as float64, exact (pg/rng.py:53-55)."""
    return draw_u32(state).astype(np.float64) * (2.0 ** -32)


# ---------------------------------------------------------------------------
# square <-> hemisphere (pg/sgmap.py:21-115)

def sq_to_dir(p):
    """Concentric square->disk then Lambert lift (pg/sgmap.py:21-33,59-65)."""
    p = np.asarray(p, dtype=np.float64)
    a = 2.0 * p[..., 0] - 1.0
    b = 2.0 * p[..., 1] - 1.0
    horiz = np.abs(a) > np.abs(b)
    a_safe = np.where(a == 0.0, 1.0, a)
    b_safe = np.where(b == 0.0, 1.0, b)
    rad = np.where(horiz, a, b)
    ang = np.where(horiz, (np.pi / 4) * (b / a_safe), (np.pi / 2) - (np.pi / 4) * (a / b_safe))
    ang = np.where((a == 0.0) & (b == 0.0), 0.0, ang)
    dx = rad * np.cos(ang)
    dy = rad * np.sin(ang)
    r2 = dx * dx + dy * dy
    lift = np.sqrt(np.maximum(2.0 - r2, 0.0))
    return np.stack([dx * lift, dy * lift, 1.0 - r2], axis=-1)


def dir_to_sq(v, check=True):
    """Inverse lift then inverse concentric map, clipped to [0,1]^2
    (pg/sgmap.py:36-56,68-77).  Raises below the hemisphere like the
    reference when ``check``."""
    v = np.asarray(v, dtype=np.float64)
    if check and np.any(v[..., 2] < -1e-9):
        raise ValueError("direction below the hemisphere (z < 0)")
    s = np.sqrt(np.maximum(1.0 + v[..., 2], 1e-30))
    x = v[..., 0] / s
    y = v[..., 1] / s
    rho = np.hypot(x, y)
    xdom = np.abs(x) >= np.abs(y)
    x_safe = np.where(x == 0.0, 1.0, x)
    y_safe = np.where(y == 0.0, 1.0, y)
    a_x = np.sign(x_safe) * rho
    b_x = np.arctan(y / x_safe) * (4.0 / np.pi) * a_x
    b_y = np.sign(y_safe) * rho
    a_y = np.arctan(x / y_safe) * (4.0 / np.pi) * b_y
    a = np.where(xdom, a_x, a_y)
    b = np.where(xdom, b_x, b_y)
    a = np.where(rho == 0.0, 0.0, a)
    b = np.where(rho == 0.0, 0.0, b)
    return np.clip(np.stack([(a + 1.0) * 0.5, (b + 1.0) * 0.5], axis=-1), 0.0, 1.0)


def onb(n):
    """Branchless revised ONB keyed on sign(n_z) (pg/sgmap.py:85-98)."""
    n = np.asarray(n, dtype=np.float64)
    nx, ny, nz = n[..., 0], n[..., 1], n[..., 2]
    sg = np.copysign(1.0, nz)
    a = -1.0 / (sg + nz)
    b = nx * ny * a
    t = np.stack([1.0 + sg * nx * nx * a, sg * b, -sg * nx], axis=-1)
    bt = np.stack([b, sg + ny * ny * a, -ny], axis=-1)
    return t, bt


def dot3(u, v):
    return np.sum(u * v, axis=-1)


def local_to_world(t, b, n, v):
    """(pg/sgmap.py:101-105)"""
    return t * v[..., 0:1] + b * v[..., 1:2] + n * v[..., 2:3]


def world_to_local(t, b, n, v):
    """(pg/sgmap.py:108-115)"""
    return np.stack([dot3(v, t), dot3(v, b), dot3(v, n)], axis=-1)


def unit(v):
    """(pg/scene.py:31-34)"""
    v = np.asarray(v, dtype=np.float64)
    return v / np.maximum(np.linalg.norm(v, axis=-1, keepdims=True), 1e-30)


# ---------------------------------------------------------------------------
# BRDFs: Lambert + GGX (alpha = r^2, separable Smith, Schlick) (pg/scene.py:247-380)

def _ndf(alpha, c):
    a2 = alpha * alpha
    d = c * c * (a2 - 1.0) + 1.0
    return a2 / np.maximum(np.pi * d * d, 1e-30)


def _g1(alpha, c):
    a2 = alpha * alpha
    return 2.0 * c / np.maximum(c + np.sqrt(a2 + (1.0 - a2) * c * c), 1e-30)


def brdf_value(kind, albedo, rough, wi, wo, n):
    """RGB BRDF (pg/scene.py:258-284)."""
    kind = np.asarray(kind)
    albedo = np.asarray(albedo, dtype=np.float64)
    ci = dot3(wi, n)
    co = dot3(wo, n)
    up = (ci > 0.0) & (co > 0.0)
    f = np.where(up[..., None], albedo / np.pi, 0.0)
    gl = kind == GLOSSY
    if np.any(gl):
        alpha = np.maximum(np.asarray(rough, dtype=np.float64) ** 2, 1e-6)
        h = unit(wi + wo)
        ch = np.abs(dot3(h, n))
        hi = dot3(h, wi)
        spec = (_ndf(alpha, ch) * (_g1(alpha, np.abs(ci)) * _g1(alpha, np.abs(co)))
                / np.maximum(4.0 * ci * co, 1e-30))
        fres = albedo + (1.0 - albedo) * np.power(np.clip(1.0 - np.abs(hi), 0.0, 1.0), 5.0)[..., None]
        f = np.where((gl & up)[..., None], fres * spec[..., None], f)
    return f


def brdf_density(kind, rough, wi, wo, n):
    """Solid-angle pdf of brdf_draw (pg/scene.py:287-308)."""
    kind = np.asarray(kind)
    ci = dot3(wi, n)
    co = dot3(wo, n)
    up = (ci > 0.0) & (co > 0.0)
    pdf = np.where(up, ci / np.pi, 0.0)
    gl = kind == GLOSSY
    if np.any(gl):
        alpha = np.maximum(np.asarray(rough, dtype=np.float64) ** 2, 1e-6)
        h = unit(wi + wo)
        ch = np.abs(dot3(h, n))
        gp = _g1(alpha, np.abs(co)) * _ndf(alpha, ch) / np.maximum(4.0 * co, 1e-30)
        pdf = np.where(gl & up, gp, pdf)
    return pdf


def _cosine_local(u1, u2):
    """(pg/scene.py:311-316)"""
    r = np.sqrt(u1)
    ang = 2.0 * np.pi * u2
    return np.stack([r * np.cos(ang), r * np.sin(ang), np.sqrt(np.maximum(1.0 - u1, 0.0))], axis=-1)


def _vndf_local(alpha, wo_l, u1, u2):
    """Heitz visible-normal GGX sampling in the local frame (pg/scene.py:319-351)."""
    a = alpha[..., None]
    vh = unit(wo_l * np.concatenate([a, a, np.ones_like(a)], axis=-1))
    l2 = vh[..., 0] ** 2 + vh[..., 1] ** 2
    ok = l2 > 1e-18
    inv = 1.0 / np.sqrt(np.where(ok, l2, 1.0))
    t1 = np.where(ok[..., None],
                  np.stack([-vh[..., 1] * inv, vh[..., 0] * inv, np.zeros_like(inv)], axis=-1),
                  np.broadcast_to(np.array([1.0, 0.0, 0.0]), vh.shape))
    t2 = np.cross(vh, t1)
    r = np.sqrt(u1)
    ph = 2.0 * np.pi * u2
    p1 = r * np.cos(ph)
    p2 = r * np.sin(ph)
    s = 0.5 * (1.0 + vh[..., 2])
    p2 = (1.0 - s) * np.sqrt(np.maximum(1.0 - p1 * p1, 0.0)) + s * p2
    nh = (p1[..., None] * t1 + p2[..., None] * t2
          + np.sqrt(np.maximum(1.0 - p1 * p1 - p2 * p2, 0.0))[..., None] * vh)
    h = unit(np.stack([alpha * nh[..., 0], alpha * nh[..., 1], np.maximum(nh[..., 2], 1e-9)], axis=-1))
    return 2.0 * np.sum(wo_l * h, axis=-1, keepdims=True) * h - wo_l


def brdf_draw(kind, rough, wo, n, state):
    """Direction, pdf, valid; consumes two draws per lane (pg/scene.py:354-380)."""
    kind = np.asarray(kind)
    u1 = draw_unit(state)
    u2 = draw_unit(state)
    t, b = onb(n)
    wl = _cosine_local(u1, u2)
    gl = kind == GLOSSY
    if np.any(gl):
        alpha = np.maximum(np.asarray(rough, dtype=np.float64) ** 2, 1e-6)
        wl = np.where(gl[..., None], _vndf_local(alpha, world_to_local(t, b, n, wo), u1, u2), wl)
    wi = local_to_world(t, b, n, wl)
    ok = (dot3(wi, n) > 1e-9) & (dot3(wo, n) > 0.0)
    pdf = brdf_density(kind, rough, wi, wo, n)
    return wi, pdf, ok & (pdf > 0.0)


def luminance(rgb):
    """(pg/scene.py:27-28)"""
    return np.asarray(rgb, dtype=np.float64) @ np.array(LUMA)


# ---------------------------------------------------------------------------
# mixture model (pg/mixture.py)

def fresh_stats(npix):
    """Initial Gamma entries (pg/mixture.py:44-59): Sigma = 0.25 I around the centre."""
    s = np.empty((npix, 8))
    s[:] = (0.5, 0.5, 0.5, 0.5, 0.25, 0.0, PI_LO, 0.0)
    return s


def chol2(sxx, sxy, syy):
    """Closed-form 2x2 Cholesky (pg/mixture.py:62-73): (l11, l21, l22)."""
    l11 = np.sqrt(sxx)
    l21 = sxy / l11
    l22 = np.sqrt(np.maximum(syy - l21 * l21, 1e-30))
    return l11, l21, l22


_GLX, _GLW = np.polynomial.legendre.leggauss(24)
_GLX = 0.5 * (_GLX + 1.0)
_GLW = 0.5 * _GLW
Z_CLIP = 8.5
RAMP = 6.5


def trunc_mass(mx, my, l11, l21, l22):
    """Mass of the Gaussian inside [0,1]^2 (pg/mixture.py:77-126).

    Whitened outer variable z in [lo1, hi1]; the inner Gaussian CDF ramps of
    the y=0 and y=1 edges saturate at +-6.5 sigma, which gives 4 break points;
    24-point Gauss-Legendre on each of the 5 sorted segments, clamped to
    [1e-4, 1]."""
    lo1 = np.maximum((0.0 - mx) / l11, -Z_CLIP)
    hi1 = np.maximum(np.minimum((1.0 - mx) / l11, Z_CLIP), lo1)
    l21s = np.where(np.abs(l21) < 1e-30, 1e-30, l21)
    brk = [np.clip(((c - my) - s * l22) / l21s, lo1, hi1) for c in (0.0, 1.0) for s in (-RAMP, RAMP)]
    edges = np.sort(np.stack(brk + [lo1, hi1], axis=-1), axis=-1)
    a = edges[..., :-1]
    ln = edges[..., 1:] - a
    z = a[..., None] + ln[..., None] * _GLX
    e = (Ellipsis, None, None)
    hi = (1.0 - my[e] - l21[e] * z) / l22[e]
    lo = (0.0 - my[e] - l21[e] * z) / l22[e]
    val = np.sum(ln[..., None] * _GLW * (np.exp(-0.5 * z * z) / np.sqrt(2.0 * np.pi)) * (ndtr(hi) - ndtr(lo)),
                 axis=(-1, -2))
    return np.clip(val, Z_FLOOR, 1.0)


def lobe(stats):
    """Gaussian lobe from Gamma moments (pg/mixture.py:129-155).

    Returns a namespace with mu (P,2), cov (P,2,2), l11, l21, l22 (P,), chol
    (P,2,2), z (P,) and the boolean ``reset`` (not part of the reference
    return, used by tests)."""
    st = np.asarray(stats, dtype=np.float64)
    mx, my = st[..., MEAN_X], st[..., MEAN_Y]
    sxx = st[..., M2_XX] - mx * mx + RIDGE
    syy = st[..., M2_YY] - my * my + RIDGE
    sxy = st[..., M2_XY] - mx * my
    half = 0.5 * (sxx + syy)
    dlt = np.sqrt(np.maximum(0.25 * (sxx - syy) ** 2 + sxy * sxy, 0.0))
    reset = (half - dlt) < EIG_FLOOR
    sxx = np.where(reset, RESET_VAR, sxx)
    syy = np.where(reset, RESET_VAR, syy)
    sxy = np.where(reset, 0.0, sxy)
    l11, l21, l22 = chol2(sxx, sxy, syy)
    cov = np.stack([np.stack([sxx, sxy], -1), np.stack([sxy, syy], -1)], -2)
    chol = np.stack([np.stack([l11, np.zeros_like(l11)], -1), np.stack([l21, l22], -1)], -2)
    z = trunc_mass(mx, my, l11, l21, l22)
    return SimpleNamespace(mu=np.stack([mx, my], -1), cov=cov, chol=chol,
                           l11=l11, l21=l21, l22=l22, z=z, reset=reset)


def gauss_sq_pdf(lb, p, sel=slice(None)):
    """Truncation-normalised density on the square (pg/mixture.py:158-169)."""
    p = np.asarray(p, dtype=np.float64)
    mu = lb.mu[sel]
    l11, l21, l22, z = lb.l11[sel], lb.l21[sel], lb.l22[sel], lb.z[sel]
    z1 = (p[..., 0] - mu[..., 0]) / l11
    z2 = ((p[..., 1] - mu[..., 1]) - l21 * z1) / l22
    return np.exp(-0.5 * (z1 * z1 + z2 * z2)) * (1.0 / (2.0 * np.pi * l11 * l22)) / z


def box_muller(u1, u2):
    """(pg/mixture.py:185-190)"""
    r = np.sqrt(-2.0 * np.log(np.maximum(u1, 1e-12)))
    ang = 2.0 * np.pi * u2
    return r * np.cos(ang), r * np.sin(ang)


def responsibility(pi, g, b):
    """E-step posterior of the Gaussian component (pg/mixture.py:262-273)."""
    num = pi * g
    den = num + (1.0 - pi) * b
    return np.where(den > 0.0, num / np.where(den > 0.0, den, 1.0), 0.0)


def budget(k, kmax=KMAX):
    """N = floor((1 - min(k,kmax)/kmax)*15 + 5 + 0.5) (pg/mixture.py:324-328)."""
    k = np.minimum(np.asarray(k, dtype=np.float64), float(kmax))
    return np.floor((1.0 - k / float(kmax)) * 15.0 + 5.0 + 0.5).astype(np.int64)


def m_step(stats, sq, w, r, ok, kmax=KMAX):
    """Online weighted M-step (pg/mixture.py:276-321), including the quirk
    that a batch with total weight > 0 but zero responsibility mass pulls
    the moments towards 0."""
    st = np.asarray(stats, dtype=np.float64)
    ok = ok & np.isfinite(w) & (w >= 0.0)
    w = np.where(ok, w, 0.0)
    r = np.where(ok, r, 0.0)
    wr = w * r
    bwr = np.sum(wr, axis=-1)
    bw = np.sum(w, axis=-1)
    x, y = sq[..., 0], sq[..., 1]
    den = np.maximum(bwr, 1e-8)
    k = st[..., EPOCH]
    eta = np.maximum(1.0 / (k + 1.0), 1.0 / float(kmax))
    out = st.copy()
    for ch, q in ((MEAN_X, x), (MEAN_Y, y), (M2_XX, x * x), (M2_YY, y * y), (M2_XY, x * y)):
        out[..., ch] = (1.0 - eta) * st[..., ch] + eta * (np.sum(wr * q, axis=-1) / den)
    out[..., MIX_PI] = np.clip((1.0 - eta) * st[..., MIX_PI] + eta * (bwr / np.maximum(bw, 1e-8)), PI_LO, PI_HI)
    out[..., W_SUM] = (1.0 - eta) * st[..., W_SUM] + eta * bwr
    out[..., EPOCH] = k + 1.0
    return np.where((bw > 0.0)[..., None], out, st)


# ---------------------------------------------------------------------------
# reprojection (pg/guide_buffers.py:78-137)

def reproject(stats_prev, prev, cur, depth_rel_tol=0.1, normal_dot_min=0.9, rotate_mean=True, return_parts=False):
    """Nearest-neighbour history fetch along motion vectors.

    stats_prev: (H,W,8) float32.  prev/cur: G-buffer namespaces (valid,
    depth, normal, pos, motion, has_history, cam_origin).  Returns (H,W,8)
    float32; with ``return_parts`` also a namespace of the per-pixel
    decisions (flat): ``source_ok`` (valid, history, in frame, source valid),
    ``gates_ok`` (+ depth and normal gates), ``accepted`` (+ mean rotation
    z >= 0)."""
    h, w = stats_prev.shape[:2]
    src_stats = stats_prev.reshape(-1, 8).astype(np.float64)
    out = fresh_stats(h * w)
    ii, jj = np.meshgrid(np.arange(h), np.arange(w), indexing="ij")
    tx = np.rint(jj + cur.motion[..., 0]).astype(np.int64)
    ty = np.rint(ii + cur.motion[..., 1]).astype(np.int64)
    ok = cur.valid & cur.has_history & (tx >= 0) & (tx < w) & (ty >= 0) & (ty < h)
    src = (np.clip(ty, 0, h - 1) * w + np.clip(tx, 0, w - 1)).reshape(-1)
    ok = ok.reshape(-1) & prev.valid.reshape(-1)[src]
    ok_src = ok.copy()
    d_exp = np.linalg.norm(cur.pos.reshape(-1, 3) - prev.cam_origin, axis=-1)
    d_prev = prev.depth.reshape(-1)[src]
    ok &= np.abs(d_prev - d_exp) < depth_rel_tol * np.maximum(d_exp, 1e-12)
    n_prev = prev.normal.reshape(-1, 3)[src]
    n_cur = cur.normal.reshape(-1, 3)
    ok &= dot3(n_prev, n_cur) > normal_dot_min
    ok_gates = ok.copy()
    sel = np.nonzero(ok)[0]
    if sel.size:
        got = src_stats[src[sel]]
        if rotate_mean:
            d_l = sq_to_dir(got[:, (MEAN_X, MEAN_Y)])
            tp, bp = onb(n_prev[sel])
            d_w = local_to_world(tp, bp, n_prev[sel], d_l)
            tc, bc = onb(n_cur[sel])
            d_c = world_to_local(tc, bc, n_cur[sel], d_w)
            keep = ~(d_c[:, 2] < 0.0)
            d_c[:, 2] = np.maximum(d_c[:, 2], 0.0)
            got[:, (MEAN_X, MEAN_Y)] = dir_to_sq(d_c)
            sel, got = sel[keep], got[keep]
        out[sel] = got
    out = out.reshape(h, w, 8).astype(np.float32)
    if return_parts:
        acc = np.zeros(h * w, dtype=bool)
        acc[sel] = True
        return out, SimpleNamespace(source_ok=ok_src, gates_ok=ok_gates, accepted=acc)
    return out


# ---------------------------------------------------------------------------
# training pass (pg/guide_buffers.py:140-231, 262-283)

def candidates(h, w, radius, state, pix=None):
    """Self + 19 uniform-disk neighbours; 38 draws per pixel, u1 block then
    u2 block (pg/guide_buffers.py:140-161).  Returns (cand, used).

    ``pix``: flat frame indices of the pixels whose candidates are drawn
    (default: every pixel); ``state`` holds their streams in that order.
    Candidates are frame indices either way."""
    pix = np.arange(h * w) if pix is None else np.asarray(pix, dtype=np.int64)
    u1 = np.stack([draw_unit(state) for _ in range(SLOTS - 1)], axis=1)
    u2 = np.stack([draw_unit(state) for _ in range(SLOTS - 1)], axis=1)
    rr = radius * np.sqrt(u1)
    ang = 2.0 * np.pi * u2
    cx = (pix % w)[:, None] + np.rint(rr * np.cos(ang)).astype(np.int64)
    cy = (pix // w)[:, None] + np.rint(rr * np.sin(ang)).astype(np.int64)
    inside = (cx >= 0) & (cx < w) & (cy >= 0) & (cy < h)
    cand = np.concatenate([pix[:, None], np.clip(cy, 0, h - 1) * w + np.clip(cx, 0, w - 1)], axis=1)
    used = np.concatenate([np.ones((pix.size, 1), dtype=bool), inside], axis=1)
    return cand, used


def records(stats, lb, vpl, gbuf, cand, used, pix=None):
    """Per (pixel, slot) record: square point, luminance weight, E-step
    responsibility and validity (pg/guide_buffers.py:170-231).  ``pix``:
    frame indices of the receivers (rows of stats / lb / cand), default all."""
    p, c = cand.shape
    own = slice(None) if pix is None else np.asarray(pix, dtype=np.int64)
    x = gbuf.pos.reshape(-1, 3)[own]
    n = gbuf.normal.reshape(-1, 3)[own]
    wo = gbuf.view.reshape(-1, 3)[own]
    kind = np.broadcast_to(gbuf.kind.reshape(-1)[own][:, None], (p, c))
    rough = np.broadcast_to(gbuf.roughness.reshape(-1)[own][:, None], (p, c))
    alb = np.broadcast_to(gbuf.albedo.reshape(-1, 3)[own][:, None, :], (p, c, 3))
    ok = used & vpl.valid.reshape(-1)[cand] & (vpl.strategy.reshape(-1)[cand] == STRAT_BRDF)
    ok &= gbuf.valid.reshape(-1)[own][:, None]
    d = vpl.y.reshape(-1, 3)[cand] - x[:, None, :]
    dist = np.linalg.norm(d, axis=-1)
    ok &= dist > 1e-9
    om = d / np.maximum(dist, 1e-12)[..., None]
    cr = dot3(om, n[:, None, :])
    ok &= cr > 1e-9
    f = brdf_value(kind, alb, rough, om, wo[:, None, :], n[:, None, :])
    wgt = luminance(vpl.radiance.reshape(-1, 3)[cand] * f * np.maximum(cr, 0.0)[..., None])
    wgt = np.where(ok, wgt, 0.0)
    t, b = onb(n)
    dl = world_to_local(t[:, None, :], b[:, None, :], n[:, None, :], om)
    dl[..., 2] = np.maximum(dl[..., 2], 0.0)
    dl = np.where(ok[..., None], dl, np.array([0.0, 0.0, 1.0]))
    sq = dir_to_sq(dl)
    lbc = SimpleNamespace(mu=lb.mu[:, None, :], l11=lb.l11[:, None], l21=lb.l21[:, None],
                          l22=lb.l22[:, None], z=lb.z[:, None])
    g = gauss_sq_pdf(lbc, sq) / (2.0 * np.pi)
    bp = brdf_density(kind, rough, om, wo[:, None, :], n[:, None, :])
    r = responsibility(stats[:, MIX_PI][:, None], g, bp)
    return sq, wgt, r, ok


def train(stats_f32, vpl, gbuf, kmax=KMAX, seed=0, frame=0, radius=RADIUS, return_parts=False, rows=None):
    """One EM epoch per valid pixel over the screen-space VPL neighbourhood
    (pg/guide_buffers.py:262-283).  Returns (H,W,8) float32.

    ``rows=(r0, r1)`` trains only frame rows r0..r1-1 (returns those rows),
    with the whole frame as context: global pixel indices key the streams
    and the in-frame test uses the full height, so the band equals the same
    rows of the whole-frame result (the reference's per-pixel independence,
    pg/guide_buffers.py:274)."""
    h, w = stats_f32.shape[:2]
    r0, r1 = (0, h) if rows is None else rows
    pix = np.arange(r0 * w, r1 * w, dtype=np.int64)
    st = stats_f32.reshape(-1, 8)[pix].astype(np.float64)
    lb = lobe(st)
    state = seed_lanes(seed, frame, pix, stream=1)
    cand, used = candidates(h, w, radius, state, pix)
    used &= np.arange(SLOTS)[None, :] < budget(st[:, EPOCH], kmax)[:, None]
    sq, wgt, r, ok = records(st, lb, vpl, gbuf, cand, used, pix)
    new = m_step(st, sq, wgt, r, ok, kmax)
    keep = ~gbuf.valid.reshape(-1)[pix]
    new[keep] = st[keep]
    out = new.reshape(r1 - r0, w, 8).astype(np.float32)
    if return_parts:
        return out, SimpleNamespace(cand=cand, used=used, sq=sq, w=wgt, r=r, ok=ok, lobe=lb)
    return out


# ---------------------------------------------------------------------------
# guided first-bounce sampling (pg/mixture.py:193-259, pg/ptrace.py:161-220)

def draw_mixture(stats, lb, kind, rough, wo_l, state):
    """One-sample mixture draw in the local frame (pg/mixture.py:193-259)
    with the BRDF callbacks of pg/ptrace.py:201-208 (normal = e_z).
    Mutates ``state``.  Returns (dir_l, pdf, strategy, valid)."""
    n = stats.shape[0]
    pi = stats[:, MIX_PI]
    gauss = draw_unit(state) < pi
    sq = np.zeros((n, 2))
    hit = np.zeros(n, dtype=bool)
    todo = np.nonzero(gauss)[0]
    for _ in range(GAUSS_TRIES):
        if todo.size == 0:
            break
        sub = state[todo]
        u1 = draw_unit(sub)
        u2 = draw_unit(sub)
        state[todo] = sub
        g0, g1 = box_muller(u1, u2)
        px = lb.mu[todo, 0] + lb.l11[todo] * g0
        py = lb.mu[todo, 1] + lb.l21[todo] * g0 + lb.l22[todo] * g1
        inside = (px >= 0.0) & (px <= 1.0) & (py >= 0.0) & (py <= 1.0)
        acc = todo[inside]
        sq[acc, 0] = px[inside]
        sq[acc, 1] = py[inside]
        hit[acc] = True
        todo = todo[~inside]
    d = np.zeros((n, 3))
    d[hit] = sq_to_dir(sq[hit])
    valid = np.ones(n, dtype=bool)
    fb = np.nonzero(~hit)[0]
    ez = np.array([0.0, 0.0, 1.0])
    if fb.size:
        sub = state[fb]
        wl, _, okb = brdf_draw(kind[fb], rough[fb], wo_l[fb], np.broadcast_to(ez, (fb.size, 3)), sub)
        state[fb] = sub
        d[fb] = wl
        valid[fb] = okb
    pdf = np.zeros(n)
    vi = np.nonzero(valid)[0]
    if vi.size:
        bp = brdf_density(kind[vi], rough[vi], d[vi], wo_l[vi], np.broadcast_to(ez, (vi.size, 3)))
        g = gauss_sq_pdf(lb, dir_to_sq(d[vi]), sel=vi) / (2.0 * np.pi)
        pdf[vi] = pi[vi] * g + (1.0 - pi[vi]) * bp
    return d, pdf, np.where(hit, STRAT_GAUSS, STRAT_BRDF).astype(np.uint8), valid


def first_bounce(pos, nrm, kind, rough, wo, stats, lb, guided, state):
    """Depth-0 scatter direction per lane (pg/ptrace.py:161-220): plain
    lanes use world-space BRDF sampling, guided lanes the local mixture.
    Mutates ``state``.  Returns (wi, pdf, strategy, valid)."""
    m = len(guided)
    wi = np.zeros((m, 3))
    pdf = np.zeros(m)
    strat = np.zeros(m, dtype=np.uint8)
    valid = np.zeros(m, dtype=bool)
    pl = np.nonzero(~guided)[0]
    if pl.size:
        sub = state[pl]
        w_, p_, ok_ = brdf_draw(kind[pl], rough[pl], wo[pl], nrm[pl], sub)
        state[pl] = sub
        wi[pl], pdf[pl], valid[pl] = w_, p_, ok_
    gs = np.nonzero(guided)[0]
    if gs.size:
        t, b = onb(nrm[gs])
        wol = world_to_local(t, b, nrm[gs], wo[gs])
        sub = state[gs]
        lbg = SimpleNamespace(mu=lb.mu[gs], l11=lb.l11[gs], l21=lb.l21[gs], l22=lb.l22[gs], z=lb.z[gs])
        dl, p_, s_, ok_ = draw_mixture(stats[gs], lbg, kind[gs], rough[gs], wol, sub)
        state[gs] = sub
        wi[gs] = local_to_world(t, b, nrm[gs], dl)
        pdf[gs] = p_
        strat[gs] = s_
        valid[gs] = ok_ & (p_ > 0.0)
    return wi, pdf, strat, valid


def sample_frame(stats_f32, gbuf, seed, frame, spp=1, nee_draws=3, rough_min=ROUGH_MIN_GUIDE, lb=None, rows=None):
    """Depth-0 sampling of every valid pixel x spp lane, as the render pass
    issues it (pg/ptrace.py:449-475, 254-291): lane key pix*spp+s,
    ``nee_draws`` draws consumed by next-event estimation first, guided iff
    valid & (diffuse | rough >= rough_min) & k >= 1.

    Returns dict with wi (P,spp,3), pdf (P,spp), strategy (P,spp) uint8,
    valid (P,spp) bool, draws (P,spp) = PCG32 draws the sampler consumed
    after the NEE draws; invalid pixels are all zero.

    ``rows=(r0, r1)``: only frame rows r0..r1-1 (P = (r1-r0) W, lane keys
    stay global)."""
    h, w = stats_f32.shape[:2]
    r0, r1 = (0, h) if rows is None else rows
    band = slice(r0 * w, r1 * w)
    p = (r1 - r0) * w
    st = stats_f32.reshape(-1, 8)[band].astype(np.float64)
    if lb is None:
        lb = lobe(st)
    valid = gbuf.valid.reshape(-1)[band]
    kind = gbuf.kind.reshape(-1)[band]
    rough = gbuf.roughness.reshape(-1)[band]
    guided = valid & ((kind == DIFFUSE) | (rough >= rough_min)) & (st[:, EPOCH] >= 1.0)
    pix = np.nonzero(valid)[0]
    out = dict(wi=np.zeros((p, spp, 3)), pdf=np.zeros((p, spp)),
               strategy=np.zeros((p, spp), dtype=np.uint8), valid=np.zeros((p, spp), dtype=bool))
    if pix.size == 0:
        return out
    pos = gbuf.pos.reshape(-1, 3)[band][pix]
    nrm = gbuf.normal.reshape(-1, 3)[band][pix]
    wo = gbuf.view.reshape(-1, 3)[band][pix]
    lbp = SimpleNamespace(mu=lb.mu[pix], l11=lb.l11[pix], l21=lb.l21[pix], l22=lb.l22[pix], z=lb.z[pix])
    out["draws"] = np.zeros((p, spp), dtype=np.int64)
    gpix = (pix + r0 * w).astype(np.uint64)
    for s in range(spp):
        state = seed_lanes(seed, frame, gpix * np.uint64(spp) + np.uint64(s), 0)
        for _ in range(nee_draws):
            draw_u32(state)
        start = state.copy()
        wi, pdf, strat, ok = first_bounce(pos, nrm, kind[pix], rough[pix], wo, st[pix], lbp, guided[pix], state)
        out["draws"][pix, s] = lcg_distance(start, state)
        out["wi"][pix, s] = wi
        out["pdf"][pix, s] = pdf
        out["strategy"][pix, s] = strat
        out["valid"][pix, s] = ok
    return out


def guiding_frame(stats_prev_f32, gbuf_prev, gbuf, vpl, seed, frame, spp=1, nee_draws=3, kmax=KMAX,
                  radius=RADIUS, depth_rel_tol=0.1, normal_dot_min=0.9, rough_min=ROUGH_MIN_GUIDE, rows=None,
                  rotate_mean=True):
    """One full guiding pass in reference order: reproject (if history),
    depth-0 sampling on the reprojected Gamma, EM on the same Gamma with the
    frame's VPLs (pg/cli.py:114-142).  Returns (gamma_reproj, samples, gamma_trained).

    ``rows=(r0, r1)``: outputs for frame rows r0..r1-1 only, the whole frame
    as context (reprojection runs over the whole frame: it is cheap)."""
    if gbuf_prev is None:
        g = stats_prev_f32
    else:
        g = reproject(stats_prev_f32, gbuf_prev, gbuf, depth_rel_tol, normal_dot_min, rotate_mean)
    smp = sample_frame(g, gbuf, seed, frame, spp, nee_draws, rough_min, rows=rows)
    g2 = train(g, vpl, gbuf, kmax, seed, frame, radius, rows=rows)
    if rows is not None:
        g = g[rows[0]:rows[1]]
    return g, smp, g2
