"""CPU oracle for the render pass that produces the guiding pass's inputs
(SURVEY.md 8f rank 1): primary-ray G-buffer, camera motion vectors, and the
path-traced lanes with next-event estimation that write the image and the
per-pixel VPLs (pg/ptrace.py:97-150, 223-355, 379-586; pg/scene.py:158-241,
386-414).

TEST INFRASTRUCTURE ONLY, like pgg_oracle.py: imported by tests/ as the
checker and by nothing in the product package.  float64 NumPy, vectorised
over lanes, restated from the reference's algorithm; pinned against the
reference's own outputs in tests/golden/render_*.npz
(tests/golden/make_golden_render.py runs the reference in the build
container).
"""

from types import SimpleNamespace

import numpy as np

from oracle.pgg_oracle import (DIFFUSE, EPOCH, ROUGH_MIN_GUIDE, STRAT_BRDF, brdf_draw, brdf_value, dot3,
                               draw_unit, first_bounce, lobe, seed_lanes)

RAY_EPS = 1e-4
LUMA = np.array([0.2126, 0.7152, 0.0722])
MAX_LANES = 1 << 18  # pg/ptrace.py:379 (lanes per batch; sets the spp chunking of the sum)


# ---------------------------------------------------------------------------
# geometry (pg/scene.py:158-241)

def cast(scene, o, d, t_min=RAY_EPS, t_max=np.inf):
    """Nearest hit of each ray over all spheres then all quads; strict
    t < best keeps the first primitive on ties (pg/scene.py:158-235).
    Returns hit, t, pos, normal (against the ray), mat, front."""
    n = o.shape[0]
    best = np.full(n, np.inf)
    which = np.full(n, -1, dtype=np.int8)
    prim = np.full(n, -1, dtype=np.int32)
    t_max = np.broadcast_to(np.asarray(t_max, dtype=np.float64), (n,))
    for i in range(len(scene.sph_radius)):
        oc = o - scene.sph_center[i]
        b = np.sum(oc * d, axis=-1)
        c = np.sum(oc * oc, axis=-1) - scene.sph_radius[i] ** 2
        disc = b * b - c
        ok = disc > 0.0
        root = np.sqrt(np.where(ok, disc, 0.0))
        near, far = -b - root, -b + root
        t = np.where((near > t_min) & (near < t_max), near, far)
        ok &= (t > t_min) & (t < t_max) & (t < best)
        best = np.where(ok, t, best)
        which = np.where(ok, 0, which)
        prim = np.where(ok, i, prim)
    for i in range(len(scene.quad_mat)):
        qn = scene.quad_normal[i]
        den = d @ qn
        ok = np.abs(den) > 1e-12
        t = np.where(ok, ((scene.quad_corner[i] - o) @ qn) / np.where(ok, den, 1.0), np.inf)
        rel = o + t[:, None] * d - scene.quad_corner[i]
        eu, ev = scene.quad_eu[i], scene.quad_ev[i]
        u = (rel @ eu) / (eu @ eu)
        v = (rel @ ev) / (ev @ ev)
        ok &= (u >= 0.0) & (u <= 1.0) & (v >= 0.0) & (v <= 1.0)
        ok &= (t > t_min) & (t < t_max) & (t < best)
        best = np.where(ok, t, best)
        which = np.where(ok, 1, which)
        prim = np.where(ok, i, prim)
    hit = which >= 0
    pos = o + best[:, None] * d
    nrm = np.zeros((n, 3))
    mat = np.full(n, -1, dtype=np.int32)
    s = hit & (which == 0)
    if np.any(s):
        k = prim[s]
        nrm[s] = (pos[s] - scene.sph_center[k]) / scene.sph_radius[k][:, None]
        mat[s] = scene.sph_mat[k]
    q = hit & (which == 1)
    if np.any(q):
        k = prim[q]
        nrm[q] = scene.quad_normal[k]
        mat[q] = scene.quad_mat[k]
    facing = np.sum(nrm * d, axis=-1)
    nrm = np.where((facing > 0.0)[:, None], -nrm, nrm)
    return SimpleNamespace(hit=hit, t=np.where(hit, best, np.inf), pos=pos, normal=nrm, mat=mat,
                           front=hit & (facing < 0.0))


def blocked(scene, o, d, t_max):
    """Any geometry inside (RAY_EPS, t_max) (pg/scene.py:238-241)."""
    return cast(scene, o, d, RAY_EPS, t_max).hit


def light_sample(scene, p, state):
    """NEE toward one uniformly picked one-sided quad emitter; three draws
    (pick, u1, u2) per lane (pg/scene.py:386-414).  Returns dir, dist, Le, pdf_sr."""
    ne = scene.num_emitters
    u_pick = draw_unit(state)
    u1 = draw_unit(state)
    u2 = draw_unit(state)
    qi = scene.emitter_quads[np.minimum((u_pick * ne).astype(np.int64), ne - 1)]
    y = scene.quad_corner[qi] + u1[:, None] * scene.quad_eu[qi] + u2[:, None] * scene.quad_ev[qi]
    d = y - p
    dist = np.maximum(np.linalg.norm(d, axis=-1), 1e-12)
    w = d / dist[:, None]
    cos_l = -np.sum(w * scene.quad_normal[qi], axis=-1)
    lit = cos_l > 1e-9
    pdf = np.where(lit, dist * dist / (scene.quad_area[qi] * np.maximum(cos_l, 1e-12) * ne), 0.0)
    le = np.where(lit[:, None], scene.mat_emission[scene.quad_mat[qi]], 0.0)
    return w, dist, le, pdf


# ---------------------------------------------------------------------------
# camera rays and the G-buffer (pg/scene.py:125-151, pg/ptrace.py:97-150)

def eye_rays(cam, w, h, px, py):
    aspect = w / float(h)
    sx = (2.0 * (px + 0.5) / w - 1.0) * cam.tan_half_fov * aspect
    sy = (1.0 - 2.0 * (py + 0.5) / h) * cam.tan_half_fov
    d = cam.forward + sx[..., None] * cam.right + sy[..., None] * cam.up
    return d / np.maximum(np.linalg.norm(d, axis=-1, keepdims=True), 1e-30)


def to_pixels(cam, w, h, pts):
    aspect = w / float(h)
    d = np.asarray(pts, dtype=np.float64) - cam.origin
    zc = d @ cam.forward
    front = zc > 1e-9
    z = np.where(front, zc, 1.0)
    xc = (d @ cam.right) / z
    yc = (d @ cam.up) / z
    return (xc / (cam.tan_half_fov * aspect) + 1.0) * 0.5 * w - 0.5, (1.0 - yc / cam.tan_half_fov) * 0.5 * h - 0.5, front


def gbuffer(scene, cam, w, h):
    """Primary hit per pixel centre (pg/ptrace.py:97-129): float64 fields
    named as the reference GBuffer; motion/has_history zero."""
    py, px = np.meshgrid(np.arange(h, dtype=np.float64), np.arange(w, dtype=np.float64), indexing="ij")
    d = eye_rays(cam, w, h, px, py).reshape(-1, 3)
    r = cast(scene, np.broadcast_to(cam.origin, d.shape), d)
    m = np.maximum(r.mat, 0)
    g = lambda a, c=None: a.reshape((h, w) if c is None else (h, w, c))  # noqa: E731
    return SimpleNamespace(
        width=w, height=h, valid=g(r.hit), pos=g(r.pos, 3), normal=g(r.normal, 3), depth=g(np.where(r.hit, r.t, 0.0)),
        mat=g(r.mat), kind=g(np.where(r.hit, scene.mat_kind[m], 0).astype(np.int32)),
        albedo=g(np.where(r.hit[:, None], scene.mat_albedo[m], 0.0), 3),
        roughness=g(np.where(r.hit, scene.mat_rough[m], 0.0)), front=g(r.front), view=g(-d, 3),
        motion=np.zeros((h, w, 2)), has_history=np.zeros((h, w), dtype=bool), cam_origin=cam.origin.copy())


def motion(prev_cam, gb):
    """Screen offsets to the previous camera's projection (pg/ptrace.py:132-150)."""
    h, w = gb.height, gb.width
    px, py, front = to_pixels(prev_cam, w, h, gb.pos.reshape(-1, 3))
    px, py = px.reshape(h, w), py.reshape(h, w)
    jj, ii = np.meshgrid(np.arange(w), np.arange(h))
    tx, ty = np.rint(px), np.rint(py)
    has = gb.valid & front.reshape(h, w) & (tx >= 0) & (tx < w) & (ty >= 0) & (ty < h)
    return np.stack([np.where(has, px - jj, 0.0), np.where(has, py - ii, 0.0)], axis=-1), has


# ---------------------------------------------------------------------------
# path lanes (pg/ptrace.py:223-355)

def trace(scene, max_depth, nee, state, valid0, pos0, nrm0, mat0, front0, view0, guide=None):
    """One path sample per lane.  ``guide`` = (stats, lobe, guided mask) turns
    on the mixture at depth 0.  Returns L, Li, vpl (valid, y, strategy), segments."""
    n = len(valid0)
    L = np.zeros((n, 3))
    Li = np.zeros((n, 3))
    v_ok = np.zeros(n, dtype=bool)
    v_y = np.zeros((n, 3))
    v_s = np.zeros(n, dtype=np.uint8)
    L[~valid0] = scene.background
    e0 = valid0 & front0
    L[e0] += scene.mat_emission[mat0[e0]]
    pos, nrm, mat, wo = pos0.copy(), nrm0.copy(), mat0.copy(), view0.copy()
    T = np.zeros((n, 3))
    T[valid0] = 1.0
    Tr = np.zeros((n, 3))
    alive = valid0.copy()
    segs = 0
    do_nee = nee and scene.num_emitters > 0
    for depth in range(max_depth):
        ix = np.nonzero(alive)[0]
        if ix.size == 0:
            break
        kd, alb, rg = scene.mat_kind[mat[ix]], scene.mat_albedo[mat[ix]], scene.mat_rough[mat[ix]]
        if do_nee:
            sub = state[ix]
            ld, dist, le, lpdf = light_sample(scene, pos[ix], sub)
            state[ix] = sub
            f = brdf_value(kd, alb, rg, ld, wo[ix], nrm[ix])
            cx = np.sum(ld * nrm[ix], axis=-1)
            cand = np.nonzero((lpdf > 0.0) & (cx > 0.0) & np.any(f > 0.0, axis=-1))[0]
            c = np.zeros((ix.size, 3))
            if cand.size:
                vis = cand[~blocked(scene, pos[ix[cand]], ld[cand], dist[cand] - RAY_EPS)]
                c[vis] = le[vis] * f[vis] * (cx[vis] / lpdf[vis])[:, None]
            L[ix] += T[ix] * c
            if depth >= 1:
                Li[ix] += Tr[ix] * c
        if depth == 0 and guide is not None and np.any(guide[2][ix]):
            st, lb, gm = guide
            sub = state[ix]
            lbs = SimpleNamespace(mu=lb.mu[ix], l11=lb.l11[ix], l21=lb.l21[ix], l22=lb.l22[ix], z=lb.z[ix])
            wi, pdf, strat, ok = first_bounce(pos[ix], nrm[ix], kd, rg, wo[ix], st[ix], lbs, gm[ix], sub)
            state[ix] = sub
        else:
            sub = state[ix]
            wi, pdf, ok = brdf_draw(kd, rg, wo[ix], nrm[ix], sub)
            state[ix] = sub
            strat = np.full(ix.size, STRAT_BRDF, dtype=np.uint8)
        f = brdf_value(kd, alb, rg, wi, wo[ix], nrm[ix])
        ci = np.sum(wi * nrm[ix], axis=-1)
        ok = ok & (pdf > 0.0) & (ci > 0.0)
        wgt = np.where(ok[:, None], f * (ci / np.where(ok, pdf, 1.0))[:, None], 0.0)
        T[ix] *= wgt
        if depth >= 1:
            Tr[ix] *= wgt
        alive[ix[~ok]] = False
        ix, wi, strat = ix[ok], wi[ok], strat[ok]
        if ix.size == 0:
            continue
        r = cast(scene, pos[ix], wi)
        segs += ix.size
        miss = ix[~r.hit]
        L[miss] += T[miss] * scene.background
        if depth >= 1:
            Li[miss] += Tr[miss] * scene.background
        alive[miss] = False
        hx = ix[r.hit]
        pos[hx], nrm[hx], mat[hx], wo[hx] = r.pos[r.hit], r.normal[r.hit], r.mat[r.hit], -wi[r.hit]
        if depth == 0:
            v_ok[hx] = True
            v_y[hx] = r.pos[r.hit]
            Tr[hx] = 1.0
            fr = r.front[r.hit]
            Li[hx[fr]] += scene.mat_emission[r.mat[r.hit][fr]]
            v_s[ix] = strat
    return L, Li, v_ok, v_y, v_s, segs


def render(scene, frame, seed, gb, spp=1, max_depth=4, nee=True, stats=None, rough_min=ROUGH_MIN_GUIDE,
           want_moments=False):
    """Whole-frame render (pg/ptrace.py:382-586).  ``stats``: (H, W, 8) Gamma
    for pg mode (None = pt).  Returns dict: image (H,W,3) float32, vpl_valid,
    vpl_y, vpl_radiance, vpl_strategy, segments, nonfinite, mean_path_length,
    lum_mean / lum_var when asked."""
    h, w = gb.height, gb.width
    npx = h * w
    valid = gb.valid.reshape(-1)
    pos = gb.pos.reshape(-1, 3)
    nrm = gb.normal.reshape(-1, 3)
    mat = np.maximum(gb.mat.reshape(-1), 0)
    front = gb.front.reshape(-1)
    view = gb.view.reshape(-1, 3)
    guide = None
    if stats is not None:
        st = np.asarray(stats, dtype=np.float64).reshape(npx, 8)
        kind = gb.kind.reshape(-1)
        gm = valid & ((kind == DIFFUSE) | (gb.roughness.reshape(-1) >= rough_min)) & (st[:, EPOCH] >= 1.0)
        guide = (st, lobe(st), gm)
    k_chunk = max(1, min(spp, MAX_LANES // max(npx, 1)))
    acc = np.zeros((npx, 3))
    lsum = np.zeros(npx)
    lsq = np.zeros(npx)
    nonfinite = segs = 0
    pix = np.arange(npx, dtype=np.int64)
    done = 0
    while done < spp:
        k = min(k_chunk, spp - done)
        lanes = (pix[:, None] * spp + (done + np.arange(k))[None, :]).reshape(-1)
        state = seed_lanes(seed, frame, lanes.astype(np.uint64), 0)
        rep = lambda a: np.repeat(a, k, axis=0)  # noqa: E731
        g = None
        if guide is not None:
            lb = guide[1]
            g = (rep(guide[0]), SimpleNamespace(mu=rep(lb.mu), l11=rep(lb.l11), l21=rep(lb.l21), l22=rep(lb.l22),
                                                z=rep(lb.z)), rep(guide[2]))
        L, Li, vv, vy, vs, sg = trace(scene, max_depth, nee, state, rep(valid), rep(pos), rep(nrm), rep(mat),
                                      rep(front), rep(view), g)
        segs += sg
        bad = ~np.all(np.isfinite(L), axis=-1)
        nonfinite += int(bad.sum())
        L[bad] = 0.0
        bad_i = ~np.all(np.isfinite(Li), axis=-1)
        Li[bad_i] = 0.0
        vv[bad_i] = False
        acc += L.reshape(npx, k, 3).sum(axis=1)
        lum = (L @ LUMA).reshape(npx, k)
        lsum += lum.sum(axis=1)
        lsq += (lum * lum).sum(axis=1)
        last = lambda a: a.reshape((npx, k) + a.shape[1:])[:, -1]  # noqa: E731
        vpl = (last(vv).copy(), last(vy).copy(), last(Li).copy(), last(vs).copy())
        done += k
    out = dict(image=(acc.reshape(h, w, 3) / spp).astype(np.float32), vpl_valid=vpl[0].reshape(h, w),
               vpl_y=vpl[1].reshape(h, w, 3), vpl_radiance=vpl[2].reshape(h, w, 3),
               vpl_strategy=vpl[3].reshape(h, w), segments=segs, nonfinite=nonfinite,
               mean_path_length=1.0 + segs / max(npx * spp, 1))
    if want_moments:
        m = lsum / spp
        out["lum_mean"] = m.reshape(h, w)
        out["lum_var"] = (np.maximum(lsq / spp - m * m, 0.0) * (spp / max(spp - 1.0, 1.0))).reshape(h, w)
    return out
