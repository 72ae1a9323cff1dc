"""Seeded synthetic workload for the guiding pass.

A static analytic scene (a holed back wall = planar tiles, a jittered grid
of spheres in front of it = curved tiles and disocclusion edges) seen by a
pinhole camera panning about (-1.37, +0.61) px/frame at wall depth.  The
G-buffer fields and the VPL buffer use the reference field names
(pg/ptrace.py:42-73); motion vectors are the previous camera's projection of
the current hit point, as pg/ptrace.py:132-150 computes them.

Everything is generated in float32 with torch so the same code runs on the
CPU (parity tests: the oracle gets exactly these values upcast to f64) and
on the GPU (bench: 1080p..8K sequences without a host round trip).  The
geometry uses only IEEE-exact ops (+ - * / sqrt, floor) so CPU and GPU
G-buffers are bitwise identical; the VPL randomness comes from a torch
Generator on the target device.
"""

from dataclasses import dataclass

import torch

TAN_HALF_FOV = 0.7
WALL_Z = 8.0
PAN_PX = (-1.37, 0.61)          # motion (du, dv) of wall pixels per frame
N_MATERIALS = 64
DIFFUSE, GLOSSY = 0, 1
STRAT_BRDF, STRAT_GAUSS = 0, 1


@dataclass
class Camera:
    origin: tuple   # float64 world position
    tan_half_fov: float = TAN_HALF_FOV


def camera_at(width, height, frame):
    """Camera translates in x/y so wall points move PAN_PX px per frame."""
    aspect = width / float(height)
    px_world = 2.0 * TAN_HALF_FOV * aspect * WALL_Z / width     # world units per px at the wall
    py_world = 2.0 * TAN_HALF_FOV * WALL_Z / height
    # wall content moves +x in the image when the camera moves -x; motion
    # (prev - cur) = -(image velocity)
    return Camera((PAN_PX[0] * px_world * frame, -PAN_PX[1] * py_world * frame, 0.0))


def _materials(seed, device):
    g = torch.Generator(device="cpu").manual_seed(0x5EED0000 + seed)
    u = torch.rand(N_MATERIALS, generator=g)
    kind = torch.where(u < 1.0 / 3.0, GLOSSY, DIFFUSE).to(torch.int32)
    rough = 0.05 + 0.95 * torch.rand(N_MATERIALS, generator=g)
    albedo = 0.2 + 0.7 * torch.rand(N_MATERIALS, 3, generator=g)
    return kind.to(device), rough.to(device), albedo.to(device)


def materials(seed=0, device="cpu"):
    """The workload's material table: (kind int32, roughness, albedo rgb) per
    material id -- what the G-buffer's kind / roughness / albedo look up."""
    return _materials(seed, device)


def _spheres(seed):
    g = torch.Generator(device="cpu").manual_seed(0x5F3E0000 + seed)
    cs, rs = [], []
    for iy in range(-2, 3):
        for ix in range(-4, 5):
            j = torch.rand(4, generator=g)
            cx = ix * 2.7 + (j[0].item() - 0.5) * 0.8
            cy = iy * 2.6 + (j[1].item() - 0.5) * 0.8
            cz = 4.6 + 1.4 * j[2].item()
            r = 0.75 + 0.45 * j[3].item()
            cs.append((cx, cy, cz))
            rs.append(r)
    return cs, rs


def gbuffer(width, height, frame, seed=0, device="cpu"):
    """Primary-hit G-buffer of frame ``frame`` (dict of float32/bool/int tensors)."""
    cam = camera_at(width, height, frame)
    f32 = torch.float32
    aspect = width / float(height)
    py, px = torch.meshgrid(torch.arange(height, device=device, dtype=f32),
                            torch.arange(width, device=device, dtype=f32), indexing="ij")
    ndc_x = (2.0 * (px + 0.5) / width - 1.0) * (TAN_HALF_FOV * aspect)
    ndc_y = (1.0 - 2.0 * (py + 0.5) / height) * TAN_HALF_FOV
    d = torch.stack([ndc_x, ndc_y, torch.ones_like(ndc_x)], dim=-1)
    d = d / torch.sqrt((d * d).sum(-1, keepdim=True))
    o = torch.tensor(cam.origin, dtype=f32, device=device)

    kinds, roughs, albedos = _materials(seed, device)
    inf = torch.full((height, width), float("inf"), device=device, dtype=f32)
    best_t = inf.clone()
    best_n = torch.zeros(height, width, 3, device=device, dtype=f32)
    best_m = torch.zeros(height, width, dtype=torch.int64, device=device)

    # back wall z = WALL_Z, normal (0,0,-1), holes on a world-space lattice
    t_w = (WALL_Z - o[2]) / d[..., 2]
    hp = o + t_w[..., None] * d
    cu = torch.floor(hp[..., 0] / 1.3).to(torch.int64)
    cv = torch.floor(hp[..., 1] / 1.1).to(torch.int64)
    hole = torch.remainder(cu + cv, 5) == 0
    wall_ok = (t_w > 1e-4) & ~hole
    best_t = torch.where(wall_ok, t_w, best_t)
    best_n[..., 2] = torch.where(wall_ok, -1.0, 0.0)
    cell = torch.floor(hp[..., 0] / 0.9).to(torch.int64) * 73856093 ^ torch.floor(hp[..., 1] / 0.9).to(torch.int64) * 19349663
    best_m = torch.where(wall_ok, torch.remainder(cell, N_MATERIALS), best_m)

    centers, radii = _spheres(seed)
    for i, (c, r) in enumerate(zip(centers, radii)):
        ct = torch.tensor(c, dtype=f32, device=device)
        oc = o - ct
        b = (d * oc).sum(-1)
        cc = (oc * oc).sum() - r * r
        disc = b * b - cc
        ok = disc > 0.0
        t0 = -b - torch.sqrt(torch.clamp(disc, min=0.0))
        ok = ok & (t0 > 1e-4) & (t0 < best_t)
        best_t = torch.where(ok, t0, best_t)
        hpos = o + t0[..., None] * d
        nrm = (hpos - ct) / r
        best_n = torch.where(ok[..., None], nrm, best_n)
        best_m = torch.where(ok, torch.tensor((i * 7 + 3) % N_MATERIALS, device=device), best_m)

    valid = torch.isfinite(best_t)
    t = torch.where(valid, best_t, torch.zeros_like(best_t))
    pos = torch.where(valid[..., None], o + t[..., None] * d, torch.zeros_like(d))
    nrm = best_n / torch.clamp(torch.sqrt((best_n * best_n).sum(-1, keepdim=True)), min=1e-30)
    nrm = torch.where(valid[..., None], nrm, torch.zeros_like(nrm))
    mat = torch.where(valid, best_m, torch.full_like(best_m, -1))
    sm = torch.clamp(mat, min=0)
    return dict(
        width=width, height=height,
        valid=valid, pos=pos, normal=nrm, depth=t,
        mat=mat.to(torch.int32),
        kind=torch.where(valid, kinds[sm], 0).to(torch.int32),
        albedo=torch.where(valid[..., None], albedos[sm], 0.0),
        roughness=torch.where(valid, roughs[sm], 0.0),
        front=valid.clone(),
        view=-d,
        motion=torch.zeros(height, width, 2, device=device, dtype=f32),
        has_history=torch.zeros(height, width, dtype=torch.bool, device=device),
        cam_origin=cam.origin,
    )


def attach_motion(gb, prev_cam_origin):
    """Motion vectors to the previous camera (pg/ptrace.py:132-150)."""
    h, w = gb["height"], gb["width"]
    f32 = torch.float32
    dev = gb["pos"].device
    aspect = w / float(h)
    o = torch.tensor(prev_cam_origin, dtype=f32, device=dev)
    dd = gb["pos"] - o
    zc = dd[..., 2]
    front = zc > 1e-9
    sz = torch.where(front, zc, torch.ones_like(zc))
    xc = dd[..., 0] / sz
    yc = dd[..., 1] / sz
    ppx = (xc / (TAN_HALF_FOV * aspect) + 1.0) * 0.5 * w - 0.5
    ppy = (1.0 - yc / TAN_HALF_FOV) * 0.5 * h - 0.5
    ii, jj = torch.meshgrid(torch.arange(h, device=dev, dtype=f32), torch.arange(w, device=dev, dtype=f32),
                            indexing="ij")
    tx = torch.round(ppx)
    ty = torch.round(ppy)
    inside = (tx >= 0) & (tx < w) & (ty >= 0) & (ty < h)
    has = gb["valid"] & front & inside
    gb["motion"] = torch.stack([torch.where(has, ppx - jj, 0.0), torch.where(has, ppy - ii, 0.0)], dim=-1)
    gb["has_history"] = has
    return gb


def vpl(gb, frame, seed=0, generator=None):
    """One VPL per pixel: valid p=0.95, BRDF strategy p=0.9,
    y = x + omega*U[0.5,3], omega 60% in a 0.15-spread world lobe and 40%
    cosine about the normal; RGB radiance Exp(0.5) x (8 in-lobe, 0.3 else)."""
    h, w = gb["height"], gb["width"]
    dev = gb["pos"].device
    f32 = torch.float32
    g = generator
    if g is None:
        g = torch.Generator(device=dev).manual_seed((seed * 1000003 + frame * 7919 + 17) & 0x7FFFFFFF)

    def U(*shape):
        return torch.rand(*shape, generator=g, device=dev, dtype=f32)

    valid = gb["valid"] & (U(h, w) < 0.95)
    strategy = torch.where(U(h, w) < 0.9, STRAT_BRDF, STRAT_GAUSS).to(torch.uint8)
    in_lobe = U(h, w) < 0.6
    ldir = torch.tensor([0.35, 0.6, -0.7], device=dev, dtype=f32)
    ldir = ldir / torch.sqrt((ldir * ldir).sum())
    lob = ldir + 0.15 * torch.randn(h, w, 3, generator=g, device=dev, dtype=f32)
    lob = lob / torch.sqrt((lob * lob).sum(-1, keepdim=True))
    # cosine lobe about the normal in a simple frame
    n = gb["normal"]
    u1, u2 = U(h, w), U(h, w)
    r = torch.sqrt(u1)
    ang = 2.0 * torch.pi * u2
    lx, ly, lz = r * torch.cos(ang), r * torch.sin(ang), torch.sqrt(torch.clamp(1.0 - u1, min=0.0))
    helper = torch.where((n[..., 0].abs() > 0.9)[..., None], torch.tensor([0.0, 1.0, 0.0], device=dev),
                         torch.tensor([1.0, 0.0, 0.0], device=dev))
    tt = torch.cross(helper, n, dim=-1)
    tt = tt / torch.clamp(torch.sqrt((tt * tt).sum(-1, keepdim=True)), min=1e-12)
    bb = torch.cross(n, tt, dim=-1)
    cosd = lx[..., None] * tt + ly[..., None] * bb + lz[..., None] * n
    om = torch.where(in_lobe[..., None], lob, cosd)
    y = gb["pos"] + om * (0.5 + 2.5 * U(h, w))[..., None]
    e = -0.5 * torch.log(torch.clamp(U(h, w, 3), min=1e-12))
    rad = e * torch.where(in_lobe, 8.0, 0.3)[..., None]
    y = torch.where(valid[..., None], y, torch.zeros_like(y))
    rad = torch.where(valid[..., None], rad, torch.zeros_like(rad))
    return dict(valid=valid, y=y, radiance=rad, strategy=strategy)


def sequence(width, height, frames, seed=0, device="cpu", first_frame=0):
    """Yield (gbuffer, vpl) per frame with motion/has_history attached from
    frame ``first_frame + 1`` on (the first frame carries no history)."""
    prev_cam = None
    for f in range(first_frame, first_frame + frames):
        gb = gbuffer(width, height, f, seed, device)
        if prev_cam is not None:
            attach_motion(gb, prev_cam)
        prev_cam = gb["cam_origin"]
        yield gb, vpl(gb, f, seed)
