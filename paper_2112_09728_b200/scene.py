"""Analytic scenes for the GPU render pass: the scene
document model of pg/scene.py (materials, spheres, quads, one-sided quad
emitters, keyframed pinhole camera) with the same loader, validation rules,
error type and built-in scenes, plus the packing of a scene into the flat
float64 table the CUDA kernels read (include/pgg.h, pgg_scene).

Geometry math runs on the device (csrc/pgg_render.cuh); the host side here
only parses documents and evaluates the camera of a frame (a handful of
float64 operations, mirroring pg/scene.py:94-151 so that primary rays and
reprojection see the same camera bits as the reference).
"""

import json
import math
from dataclasses import dataclass

import numpy as np

DIFFUSE = 0
GLOSSY = 1
LUMA_WEIGHTS = np.array([0.2126, 0.7152, 0.0722])
RAY_EPS = 1e-4  # pg/scene.py:24

# packed table layout (doubles per record), shared with pgg_render.cuh
MAT_STRIDE = 12   # kind, albedo rgb, roughness, emission rgb, albedo / pi rgb, pad
SPH_STRIDE = 8    # center xyz, radius, material, pad x3
QUAD_STRIDE = 16  # corner xyz, eu xyz, ev xyz, normal xyz, area, material, |eu|^2, |ev|^2


class SceneError(ValueError):
    """Malformed or invariant-violating scene document (pg/scene.py:37-38)."""


def luminance(rgb):
    return np.asarray(rgb, dtype=np.float64) @ LUMA_WEIGHTS


def normalize(v):
    v = np.asarray(v, dtype=np.float64)
    n = np.linalg.norm(v, axis=-1, keepdims=True)
    return v / np.maximum(n, 1e-30)


@dataclass(frozen=True)
class CameraKeyframe:
    frame: int
    origin: np.ndarray
    look_at: np.ndarray
    up: np.ndarray
    fov_deg: float


@dataclass(frozen=True)
class Camera:
    origin: np.ndarray
    forward: np.ndarray
    right: np.ndarray
    up: np.ndarray
    tan_half_fov: float


@dataclass
class Scene:
    """Struct-of-arrays scene, field for field the reference's pg/scene.py:58-83."""

    mat_names: list
    mat_kind: np.ndarray
    mat_albedo: np.ndarray
    mat_rough: np.ndarray
    mat_emission: np.ndarray
    sph_center: np.ndarray
    sph_radius: np.ndarray
    sph_mat: np.ndarray
    quad_corner: np.ndarray
    quad_eu: np.ndarray
    quad_ev: np.ndarray
    quad_normal: np.ndarray
    quad_area: np.ndarray
    quad_mat: np.ndarray
    emitter_quads: np.ndarray
    keyframes: list
    background: np.ndarray

    @property
    def num_emitters(self):
        return len(self.emitter_quads)

    def pack(self):
        """Flat float64 table: materials, spheres, quads, emitter indices
        (pgg_scene in include/pgg.h).  Returns (table, counts)."""
        nm, ns, nq, ne = len(self.mat_kind), len(self.sph_radius), len(self.quad_mat), self.num_emitters
        mats = np.zeros((nm, MAT_STRIDE))
        mats[:, 0] = self.mat_kind
        mats[:, 1:4] = self.mat_albedo
        mats[:, 4] = self.mat_rough
        mats[:, 5:8] = self.mat_emission
        mats[:, 8:11] = self.mat_albedo / np.pi  # the reference's Lambert value (pg/scene.py:268), same rounding
        sph = np.zeros((ns, SPH_STRIDE))
        if ns:
            sph[:, 0:3] = self.sph_center
            sph[:, 3] = self.sph_radius
            sph[:, 4] = self.sph_mat
        quad = np.zeros((nq, QUAD_STRIDE))
        if nq:
            quad[:, 0:3] = self.quad_corner
            quad[:, 3:6] = self.quad_eu
            quad[:, 6:9] = self.quad_ev
            quad[:, 9:12] = self.quad_normal
            quad[:, 12] = self.quad_area
            quad[:, 13] = self.quad_mat
            quad[:, 14] = np.sum(self.quad_eu * self.quad_eu, axis=-1)
            quad[:, 15] = np.sum(self.quad_ev * self.quad_ev, axis=-1)
        table = np.concatenate([mats.ravel(), sph.ravel(), quad.ravel(), self.emitter_quads.astype(np.float64)])
        return np.ascontiguousarray(table), (nm, ns, nq, ne)


# ---------------------------------------------------------------------------
# camera (pg/scene.py:94-151)

def camera_at(scene, frame_index):
    """Camera of a frame: linear interpolation between the bracketing keyframes."""
    kf = scene.keyframes
    f = float(frame_index)
    t = 0.0
    if len(kf) == 1 or f <= kf[0].frame:
        a = b = kf[0]
    elif f >= kf[-1].frame:
        a = b = kf[-1]
    else:
        j = 1
        while kf[j].frame < f:
            j += 1
        a, b = kf[j - 1], kf[j]
        t = (f - a.frame) / float(b.frame - a.frame)
    origin = (1 - t) * a.origin + t * b.origin
    look = (1 - t) * a.look_at + t * b.look_at
    up_hint = normalize((1 - t) * a.up + t * b.up)
    fov = (1 - t) * a.fov_deg + t * b.fov_deg
    fwd = normalize(look - origin)
    right = normalize(np.cross(fwd, up_hint))
    return Camera(origin, fwd, right, np.cross(right, fwd), math.tan(math.radians(fov) * 0.5))


def camera_is_static(scene):
    k0 = scene.keyframes[0]
    return all(np.array_equal(k.origin, k0.origin) and np.array_equal(k.look_at, k0.look_at)
               and np.array_equal(k.up, k0.up) and k.fov_deg == k0.fov_deg for k in scene.keyframes)


# ---------------------------------------------------------------------------
# loading and validation (pg/scene.py:418-573)

_KEYS = {
    "scene": {"materials", "primitives", "camera", "background"},
    "material": {"name", "kind", "albedo", "roughness", "emission"},
    "sphere": {"type", "center", "radius", "material"},
    "quad": {"type", "corner", "edge_u", "edge_v", "material"},
    "camera": {"frame", "origin", "look_at", "up", "fov_deg"},
}


def _vec3(value, what):
    ok = isinstance(value, (list, tuple)) and len(value) == 3 and all(isinstance(x, (int, float)) for x in value)
    if not ok:
        raise SceneError(f"{what}: expected a 3-vector, got {value!r}")
    return np.array(value, dtype=np.float64)


def _only(obj, kind, what):
    extra = set(obj) - _KEYS[kind]
    if extra:
        raise SceneError(f"{what}: unknown fields {sorted(extra)}")


def load_scene(text):
    """A built-in scene name or a JSON scene document -> Scene."""
    if text in BUILTIN_SCENES:
        return scene_from_dict(BUILTIN_SCENES[text]())
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as e:
        raise SceneError(f"scene parse error at line {e.lineno}, column {e.colno}: {e.msg}") from e
    return scene_from_dict(doc)


def _materials(doc):
    out = []
    names = {}
    for i, m in enumerate(doc["materials"]):
        what = f"material #{i} ({m.get('name', '?')})"
        _only(m, "material", what)
        name = m.get("name")
        if not isinstance(name, str) or not name:
            raise SceneError(f"{what}: missing name")
        if name in names:
            raise SceneError(f"{what}: duplicate material name")
        kind = m.get("kind", "diffuse")
        if kind not in ("diffuse", "glossy"):
            raise SceneError(f"{what}: kind must be 'diffuse' or 'glossy'")
        albedo = _vec3(m.get("albedo", [0.0, 0.0, 0.0]), what + " albedo")
        if np.any(albedo < 0.0) or np.any(albedo > 1.0):
            raise SceneError(f"{what}: albedo outside [0,1]")
        rough = float(m.get("roughness", 0.0))
        if not 0.0 <= rough <= 1.0:
            raise SceneError(f"{what}: roughness outside [0,1]")
        emission = _vec3(m.get("emission", [0.0, 0.0, 0.0]), what + " emission")
        if np.any(emission < 0.0) or not np.all(np.isfinite(emission)):
            raise SceneError(f"{what}: emission must be finite and >= 0")
        names[name] = i
        out.append((name, DIFFUSE if kind == "diffuse" else GLOSSY, albedo, rough, emission))
    return out, names


def _primitives(doc, names, emissions):
    sph, quads = [], []
    for i, p in enumerate(doc["primitives"]):
        ptype = p.get("type")
        what = f"primitive #{i} ({ptype})"
        if ptype not in ("sphere", "quad"):
            raise SceneError(f"{what}: type must be 'sphere' or 'quad'")
        _only(p, ptype, what)
        mname = p.get("material")
        if ptype == "sphere":
            c = _vec3(p.get("center"), what + " center")
            r = p.get("radius")
            if not isinstance(r, (int, float)) or r <= 0:
                raise SceneError(f"{what}: radius must be > 0")
            if mname not in names:
                raise SceneError(f"{what}: unknown material {mname!r}")
            if np.any(emissions[names[mname]] > 0):
                raise SceneError(f"{what}: emissive spheres are not supported; emitters must be quads")
            sph.append((c, float(r), names[mname]))
        else:
            corner = _vec3(p.get("corner"), what + " corner")
            eu = _vec3(p.get("edge_u"), what + " edge_u")
            ev = _vec3(p.get("edge_v"), what + " edge_v")
            if np.linalg.norm(np.cross(eu, ev)) < 1e-12:
                raise SceneError(f"{what}: degenerate quad (parallel or zero edges)")
            if mname not in names:
                raise SceneError(f"{what}: unknown material {mname!r}")
            quads.append((corner, eu, ev, names[mname]))
    return sph, quads


def _keyframes(doc):
    kfs = []
    for i, k in enumerate(doc["camera"]):
        what = f"camera keyframe #{i}"
        _only(k, "camera", what)
        fov = k.get("fov_deg")
        if not isinstance(fov, (int, float)) or not 1.0 < fov < 179.0:
            raise SceneError(f"{what}: fov_deg must lie in (1, 179)")
        origin = _vec3(k.get("origin"), what + " origin")
        look = _vec3(k.get("look_at"), what + " look_at")
        up = _vec3(k.get("up"), what + " up")
        if np.linalg.norm(look - origin) < 1e-12:
            raise SceneError(f"{what}: look_at coincides with origin")
        if np.linalg.norm(np.cross(look - origin, up)) < 1e-9:
            raise SceneError(f"{what}: up is parallel to the view direction")
        kfs.append(CameraKeyframe(int(k.get("frame", 0)), origin, look, normalize(up), float(fov)))
    return sorted(kfs, key=lambda k: k.frame)


def scene_from_dict(doc):
    if not isinstance(doc, dict):
        raise SceneError("scene document must be a JSON object")
    _only(doc, "scene", "scene")
    for key in ("materials", "primitives", "camera"):
        if not isinstance(doc.get(key), list) or not doc[key]:
            raise SceneError(f"scene: missing or empty '{key}' array")
    mats, names = _materials(doc)
    emissions = np.array([m[4] for m in mats])
    sph, quads = _primitives(doc, names, emissions)
    keyframes = _keyframes(doc)
    background = _vec3(doc.get("background", [0.0, 0.0, 0.0]), "background")
    if np.any(background < 0.0):
        raise SceneError("background must be >= 0")
    quad_mat = np.array([q[3] for q in quads], dtype=np.int32)
    emitters = np.array([i for i, m in enumerate(quad_mat) if np.any(emissions[m] > 0)], dtype=np.int32)
    if len(emitters) == 0 and not np.any(background > 0.0):
        raise SceneError("scene has no emitters and a black background")
    eu = np.array([q[1] for q in quads]).reshape(-1, 3)
    ev = np.array([q[2] for q in quads]).reshape(-1, 3)
    cr = np.cross(eu, ev) if len(quads) else np.zeros((0, 3))
    area = np.linalg.norm(cr, axis=-1) if len(quads) else np.zeros(0)
    return Scene(
        mat_names=[m[0] for m in mats],
        mat_kind=np.array([m[1] for m in mats], dtype=np.int32),
        mat_albedo=np.array([m[2] for m in mats]).reshape(-1, 3),
        mat_rough=np.array([m[3] for m in mats], dtype=np.float64),
        mat_emission=emissions.reshape(-1, 3),
        sph_center=np.array([s[0] for s in sph]).reshape(-1, 3),
        sph_radius=np.array([s[1] for s in sph], dtype=np.float64),
        sph_mat=np.array([s[2] for s in sph], dtype=np.int32),
        quad_corner=np.array([q[0] for q in quads]).reshape(-1, 3),
        quad_eu=eu,
        quad_ev=ev,
        quad_normal=cr / np.maximum(area[:, None], 1e-30) if len(quads) else np.zeros((0, 3)),
        quad_area=area,
        quad_mat=quad_mat,
        emitter_quads=emitters,
        keyframes=keyframes,
        background=background,
    )


# ---------------------------------------------------------------------------
# built-in scenes (the documents of pg/scene.py:580-706; scene data, names
# are part of the CLI surface)

def _box_walls(floor, ceil, back, front, left, right):
    """The six walls of the 2x2x2 box, inward-facing edge order."""
    return [
        {"type": "quad", "corner": [0, 0, 0], "edge_u": [0, 0, 2], "edge_v": [2, 0, 0], "material": floor},
        {"type": "quad", "corner": [0, 2, 0], "edge_u": [2, 0, 0], "edge_v": [0, 0, 2], "material": ceil},
        {"type": "quad", "corner": [0, 0, 2], "edge_u": [0, 2, 0], "edge_v": [2, 0, 0], "material": back},
        {"type": "quad", "corner": [0, 0, 0], "edge_u": [2, 0, 0], "edge_v": [0, 2, 0], "material": front},
        {"type": "quad", "corner": [0, 0, 0], "edge_u": [0, 2, 0], "edge_v": [0, 0, 2], "material": left},
        {"type": "quad", "corner": [2, 0, 0], "edge_u": [0, 0, 2], "edge_v": [0, 2, 0], "material": right},
    ]


def _mat(name, albedo, kind="diffuse", roughness=None, emission=None):
    m = {"name": name, "kind": kind, "albedo": albedo}
    if roughness is not None:
        m["roughness"] = roughness
    if emission is not None:
        m["emission"] = emission
    return m


def _cornell_occluder():
    """Closed box; a tall panel hides a small up-facing lamp, so the visible
    room is lit by one bounce off the ceiling strip behind the panel."""
    return {
        "materials": [
            _mat("white", [0.75, 0.75, 0.75]), _mat("red", [0.75, 0.25, 0.25]),
            _mat("green", [0.25, 0.75, 0.25]), _mat("panel", [0.70, 0.70, 0.70]),
            _mat("blue", [0.35, 0.35, 0.65]), _mat("lamp", [0.0, 0.0, 0.0], emission=[42.0, 38.0, 30.0]),
        ],
        "primitives": _box_walls("white", "white", "white", "white", "red", "green") + [
            {"type": "quad", "corner": [0.35, 0, 0.9], "edge_u": [1.3, 0, 0], "edge_v": [0, 1.45, 0],
             "material": "panel"},
            {"type": "quad", "corner": [0.7, 0.55, 1.0], "edge_u": [0, 0, 0.35], "edge_v": [0.6, 0, 0],
             "material": "lamp"},
            {"type": "sphere", "center": [0.55, 0.3, 0.45], "radius": 0.3, "material": "blue"},
        ],
        "camera": [{"frame": 0, "origin": [1.0, 1.0, 0.12], "look_at": [1.0, 1.0, 2.0], "up": [0, 1, 0],
                    "fov_deg": 68}],
        "background": [0.0, 0.0, 0.0],
    }


def _indirect_corridor():
    """Corridor whose baffled lamp faces away from the camera: the camera
    region only sees light through the slit above the baffle."""
    return {
        "materials": [
            _mat("wall", [0.80, 0.78, 0.74]), _mat("floor", [0.70, 0.70, 0.72]),
            _mat("lamp", [0.0, 0.0, 0.0], emission=[90.0, 85.0, 75.0]),
        ],
        "primitives": [
            {"type": "quad", "corner": [0, 0, 0], "edge_u": [0, 0, 3.2], "edge_v": [1, 0, 0], "material": "floor"},
            {"type": "quad", "corner": [0, 1, 0], "edge_u": [1, 0, 0], "edge_v": [0, 0, 3.2], "material": "wall"},
            {"type": "quad", "corner": [0, 0, 0], "edge_u": [0, 1, 0], "edge_v": [0, 0, 3.2], "material": "wall"},
            {"type": "quad", "corner": [1, 0, 0], "edge_u": [0, 0, 3.2], "edge_v": [0, 1, 0], "material": "wall"},
            {"type": "quad", "corner": [0, 0, 3.2], "edge_u": [0, 1, 0], "edge_v": [1, 0, 0], "material": "wall"},
            {"type": "quad", "corner": [0, 0, 0], "edge_u": [1, 0, 0], "edge_v": [0, 1, 0], "material": "wall"},
            {"type": "quad", "corner": [0, 0, 2.5], "edge_u": [1, 0, 0], "edge_v": [0, 0.62, 0], "material": "wall"},
            {"type": "quad", "corner": [0.2, 0.12, 2.6], "edge_u": [0.6, 0, 0], "edge_v": [0, 0.42, 0],
             "material": "lamp"},
        ],
        "camera": [{"frame": 0, "origin": [0.5, 0.5, 0.25], "look_at": [0.5, 0.45, 3.2], "up": [0, 1, 0],
                    "fov_deg": 60}],
        "background": [0.0, 0.0, 0.0],
    }


def _glossy_box():
    """Box with a GGX floor (roughness 0.2) and a ceiling lamp."""
    return {
        "materials": [
            _mat("white", [0.73, 0.73, 0.73]), _mat("red", [0.65, 0.22, 0.22]),
            _mat("green", [0.22, 0.65, 0.22]),
            _mat("metal", [0.85, 0.82, 0.75], kind="glossy", roughness=0.2),
            _mat("lamp", [0.0, 0.0, 0.0], emission=[16.0, 15.0, 13.0]),
        ],
        "primitives": _box_walls("metal", "white", "white", "white", "red", "green") + [
            {"type": "quad", "corner": [0.75, 1.999, 0.75], "edge_u": [0.5, 0, 0], "edge_v": [0, 0, 0.5],
             "material": "lamp"},
            {"type": "sphere", "center": [1.35, 0.35, 1.3], "radius": 0.35, "material": "white"},
        ],
        "camera": [{"frame": 0, "origin": [1.0, 1.0, 0.12], "look_at": [1.0, 0.9, 2.0], "up": [0, 1, 0],
                    "fov_deg": 68}],
        "background": [0.0, 0.0, 0.0],
    }


BUILTIN_SCENES = {
    "cornell-occluder": _cornell_occluder,
    "indirect-corridor": _indirect_corridor,
    "glossy-box": _glossy_box,
}


# ---------------------------------------------------------------------------
# Scene routines on the GPU (pg/scene.py:125-414), NumPy / torch in and out.
# Batch entry points of csrc/pgg_render.cu (the same float64 device code the
# render kernels use); `streams` are advanced in place like the reference's.

def _dev():
    from . import _conv
    return _conv.device()


def _d64(a, shape=None):
    import torch

    from . import _conv
    t = _conv.to_dev(a, torch.float64)
    return t.reshape(shape) if shape is not None else t


def _out(t, like_torch):
    return t if like_torch else t.cpu().numpy()


def _device_scene(scene):
    from .render import device_scene
    return device_scene(scene, _dev())


def _states_in(streams):
    import torch

    from . import _conv
    if torch.is_tensor(streams):
        return streams.view(torch.int64) if streams.is_cuda else _conv.u64_to_dev(streams)
    return _conv.u64_to_dev(np.asarray(streams))


def _states_back(streams, states):
    import torch
    if torch.is_tensor(streams):
        if not streams.is_cuda:
            streams.copy_(states.cpu().view(streams.dtype))
    else:
        streams[...] = states.cpu().numpy().view(np.uint64).reshape(np.shape(streams))


def intersect(scene, origins, dirs, t_min=RAY_EPS, t_max=np.inf):
    """Nearest hit per ray (pg/scene.py:158-235): dict hit, t, pos, normal, mat, front, is_emitter."""
    import torch

    from . import _lib
    like = torch.is_tensor(origins)
    o = _d64(origins, (-1, 3))
    d = _d64(dirs, (-1, 3))
    n = o.shape[0]
    tmin = torch.broadcast_to(_d64(t_min), (n,)).contiguous()
    tmax = torch.broadcast_to(_d64(t_max), (n,)).contiguous()
    ds = _device_scene(scene)
    hit = torch.empty(n, dtype=torch.uint8, device=o.device)
    t = torch.empty(n, dtype=torch.float64, device=o.device)
    pos = torch.empty(n, 3, dtype=torch.float64, device=o.device)
    nrm = torch.empty(n, 3, dtype=torch.float64, device=o.device)
    mat = torch.empty(n, dtype=torch.int32, device=o.device)
    front = torch.empty(n, dtype=torch.uint8, device=o.device)
    import ctypes
    _lib.check(_lib.lib().pgg_intersect(ctypes.byref(ds.abi), n, _lib.ptr(o), _lib.ptr(d), _lib.ptr(tmin),
                                        _lib.ptr(tmax), 0, _lib.ptr(hit), _lib.ptr(t), _lib.ptr(pos), _lib.ptr(nrm),
                                        _lib.ptr(mat), _lib.ptr(front), _lib.stream_ptr()))
    h = hit.bool()
    em = torch.as_tensor(np.any(scene.mat_emission > 0.0, axis=-1), device=o.device)
    is_em = h & em[mat.clamp(min=0).long()]
    out = {"hit": h, "t": t, "pos": pos, "normal": nrm, "mat": mat, "front": front.bool(), "is_emitter": is_em}
    return {k: _out(v, like) for k, v in out.items()}


def occluded(scene, origins, dirs, t_max):
    """True where geometry blocks the segment (RAY_EPS, t_max) (pg/scene.py:238-241)."""
    import ctypes

    import torch

    from . import _lib
    like = torch.is_tensor(origins)
    o = _d64(origins, (-1, 3))
    d = _d64(dirs, (-1, 3))
    n = o.shape[0]
    tmin = torch.full((n,), RAY_EPS, dtype=torch.float64, device=o.device)
    tmax = torch.broadcast_to(_d64(t_max), (n,)).contiguous()
    hit = torch.empty(n, dtype=torch.uint8, device=o.device)
    ds = _device_scene(scene)
    _lib.check(_lib.lib().pgg_intersect(ctypes.byref(ds.abi), n, _lib.ptr(o), _lib.ptr(d), _lib.ptr(tmin),
                                        _lib.ptr(tmax), 1, _lib.ptr(hit), None, None, None, None, None,
                                        _lib.stream_ptr()))
    return _out(hit.bool(), like)


def sample_emitter(scene, points, streams):
    """NEE toward one uniformly picked quad emitter (pg/scene.py:386-414);
    three draws per lane, `streams` advanced in place.  Returns (dir, dist, emitted, pdf_sr)."""
    import ctypes

    import torch

    from . import _lib
    like = torch.is_tensor(points)
    p = _d64(points, (-1, 3))
    n = p.shape[0]
    st = _states_in(streams).contiguous()
    dev = p.device
    w = torch.empty(n, 3, dtype=torch.float64, device=dev)
    dist = torch.empty(n, dtype=torch.float64, device=dev)
    le = torch.empty(n, 3, dtype=torch.float64, device=dev)
    pdf = torch.empty(n, dtype=torch.float64, device=dev)
    ds = _device_scene(scene)
    _lib.check(_lib.lib().pgg_sample_emitter(ctypes.byref(ds.abi), n, _lib.ptr(p), _lib.ptr(st), _lib.ptr(w),
                                             _lib.ptr(dist), _lib.ptr(le), _lib.ptr(pdf), _lib.stream_ptr()))
    _states_back(streams, st)
    return tuple(_out(v, like) for v in (w, dist, le, pdf))


def _brdf(op, kind, albedo, rough, wi, wo, n, streams=None):
    import torch

    from . import _conv, _lib
    like = any(torch.is_tensor(x) for x in (wi, wo, n) if x is not None)
    wo_t = _d64(wo, (-1, 3))
    m = wo_t.shape[0]
    dev = wo_t.device
    nn = torch.broadcast_to(_d64(n, (-1, 3)), (m, 3)).contiguous()
    k = torch.broadcast_to(_conv.to_dev(kind, torch.int32).reshape(-1), (m,)).contiguous()
    r = torch.broadcast_to(_d64(rough).reshape(-1), (m,)).contiguous()
    alb = torch.broadcast_to(_d64(albedo, (-1, 3)), (m, 3)).contiguous() if albedo is not None else None
    wi_t = _d64(wi, (-1, 3)).clone() if wi is not None else torch.empty(m, 3, dtype=torch.float64, device=dev)
    f = torch.empty(m, 3, dtype=torch.float64, device=dev) if op == 0 else None
    pdf = torch.empty(m, dtype=torch.float64, device=dev) if op >= 1 else None
    valid = torch.empty(m, dtype=torch.uint8, device=dev) if op == 2 else None
    st = _states_in(streams).contiguous() if op == 2 else None
    _lib.check(_lib.lib().pgg_brdf(op, m, _lib.ptr(k), _lib.ptr(alb), _lib.ptr(r), _lib.ptr(wi_t), _lib.ptr(wo_t),
                                   _lib.ptr(nn), _lib.ptr(st), _lib.ptr(f), _lib.ptr(pdf), _lib.ptr(valid),
                                   _lib.stream_ptr()))
    if op == 0:
        return _out(f, like)
    if op == 1:
        return _out(pdf, like)
    _states_back(streams, st)
    return _out(wi_t, like), _out(pdf, like), _out(valid.bool(), like)


def brdf_eval(kind, albedo, rough, wi, wo, n):
    """BRDF value (RGB), zero below the surface (pg/scene.py:258-284)."""
    return _brdf(0, kind, albedo, rough, wi, wo, n)


def brdf_pdf(kind, rough, wi, wo, n):
    """Solid-angle density of brdf_sample (pg/scene.py:287-308)."""
    return _brdf(1, kind, None, rough, wi, wo, n)


def brdf_sample(kind, albedo, rough, wo, n, streams):
    """Scatter direction, pdf, valid; two draws per lane (pg/scene.py:354-380)."""
    return _brdf(2, kind, albedo, rough, None, wo, n, streams)


def primary_ray_dirs(cam, width, height, px, py):
    """World ray directions through pixel centres (pg/scene.py:125-135)."""
    import torch

    from . import _lib
    from .render import camera_abi
    like = torch.is_tensor(px)
    shape = tuple(np.shape(px))
    x = _d64(px).reshape(-1).contiguous()
    y = torch.broadcast_to(_d64(py).reshape(shape), shape).reshape(-1).contiguous()
    out = torch.empty(x.shape[0], 3, dtype=torch.float64, device=x.device)
    import ctypes
    c = camera_abi(cam)
    _lib.check(_lib.lib().pgg_primary_rays(ctypes.byref(c), int(width), int(height), x.shape[0], _lib.ptr(x),
                                           _lib.ptr(y), _lib.ptr(out), _lib.stream_ptr()))
    return _out(out.reshape(shape + (3,)), like)


def project_to_pixels(cam, width, height, points):
    """World points -> continuous pixel coordinates (pg/scene.py:138-151): (px, py, in_front)."""
    import ctypes

    import torch

    from . import _lib
    from .render import camera_abi
    like = torch.is_tensor(points)
    p = _d64(points, (-1, 3))
    n = p.shape[0]
    px = torch.empty(n, dtype=torch.float64, device=p.device)
    py = torch.empty(n, dtype=torch.float64, device=p.device)
    fr = torch.empty(n, dtype=torch.uint8, device=p.device)
    c = camera_abi(cam)
    _lib.check(_lib.lib().pgg_project(ctypes.byref(c), int(width), int(height), n, _lib.ptr(p), _lib.ptr(px),
                                      _lib.ptr(py), _lib.ptr(fr), _lib.stream_ptr()))
    return _out(px, like), _out(py, like), _out(fr.bool(), like)
