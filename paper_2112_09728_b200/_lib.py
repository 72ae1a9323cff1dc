"""ctypes binding of libpgg.so (the C ABI declared in include/pgg.h).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).
There is no CPU implementation behind this module: if the library or a CUDA
device is missing every entry point raises ``PggUnavailable``.
"""

import ctypes
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PGG_LIB") or os.path.join(_HERE, "libpgg.so")  # PGG_LIB: A/B builds


IMAGE_ERROR_SCRATCH = 1184  # PGG_IMAGE_ERROR_SCRATCH (include/pgg.h)


class PggUnavailable(RuntimeError):
    """libpgg.so or a CUDA device is missing (there is no CPU fallback)."""


class PggError(RuntimeError):
    """A libpgg entry point returned a non-zero status."""


c_i32, c_i64, c_u64, c_f64, c_p = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p


class GBuffer(ctypes.Structure):
    _fields_ = [("flags", c_p), ("nd", c_p), ("pr", c_p), ("va", c_p), ("am", c_p), ("row0", c_i32),
                ("rows", c_i32)]


class GammaIn(ctypes.Structure):
    _fields_ = [("g0", c_p), ("g1", c_p), ("row0", c_i32), ("rows", c_i32)]


class GammaOut(ctypes.Structure):
    _fields_ = [("g0", c_p), ("g1", c_p)]


class Vpl(ctypes.Structure):
    _fields_ = [("y", c_p), ("L", c_p), ("row0", c_i32), ("rows", c_i32)]


class Samples(ctypes.Structure):
    _fields_ = [("dir", c_p), ("tag", c_p)]


class Config(ctypes.Structure):
    _fields_ = [("width", c_i32), ("height", c_i32), ("row0", c_i32), ("rows", c_i32), ("spp", c_i32),
                ("nee_draws", c_i32), ("k_max", c_i32), ("rotate_mean", c_i32), ("radius", c_f64),
                ("depth_rel_tol", c_f64), ("normal_dot_min", c_f64), ("rough_min_guide", c_f64),
                ("prev_cam", c_f64 * 3), ("key_sample", c_u64), ("key_train", c_u64)]


class Scene(ctypes.Structure):
    _fields_ = [("table", c_p), ("n_mat", c_i32), ("n_sph", c_i32), ("n_quad", c_i32), ("n_emit", c_i32),
                ("background", c_f64 * 3)]


class Camera(ctypes.Structure):
    _fields_ = [("origin", c_f64 * 3), ("forward", c_f64 * 3), ("right", c_f64 * 3), ("up", c_f64 * 3),
                ("tan_half_fov", c_f64)]


class RenderConfig(ctypes.Structure):
    _fields_ = [("width", c_i32), ("height", c_i32), ("row0", c_i32), ("rows", c_i32), ("spp", c_i32),
                ("max_depth", c_i32), ("nee", c_i32), ("reserved", c_i32), ("key", c_u64)]


class RenderOut(ctypes.Structure):
    _fields_ = [("image", c_p), ("vpl_y", c_p), ("vpl_L", c_p), ("lum_moments", c_p), ("counters", c_p),
                ("states", c_p)]


_SIGS = {
    "pgg_guiding_pass": [ctypes.POINTER(Config), ctypes.POINTER(GBuffer), ctypes.POINTER(GBuffer),
                         ctypes.POINTER(GammaIn), ctypes.POINTER(Vpl), ctypes.POINTER(GammaOut),
                         ctypes.POINTER(GammaOut), ctypes.POINTER(Samples), c_p, c_p],
    "pgg_reproject": [ctypes.POINTER(Config), ctypes.POINTER(GBuffer), ctypes.POINTER(GBuffer), ctypes.POINTER(GammaIn),
                      ctypes.POINTER(GammaOut), c_p, c_p],
    "pgg_train": [ctypes.POINTER(Config), ctypes.POINTER(GBuffer), ctypes.POINTER(GammaIn), ctypes.POINTER(Vpl),
                  ctypes.POINTER(GammaOut), c_p, c_p],
    "pgg_sample_first_bounce": [ctypes.POINTER(Config), ctypes.POINTER(GBuffer), ctypes.POINTER(GammaIn),
                                ctypes.POINTER(Samples), c_p],
    "pgg_train_records": [ctypes.POINTER(Config), ctypes.POINTER(GBuffer), ctypes.POINTER(GammaIn),
                          ctypes.POINTER(Vpl), c_i64, c_p, c_p, c_p, c_p],
    "pgg_sample_lanes": [c_i64, c_i32, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p],
    "pgg_lobe": [c_i64, c_p, c_p, c_p, c_p, c_p, c_p, c_p],
    "pgg_trunc_mass": [c_i64, c_p, c_p, c_p, c_p],
    "pgg_m_step": [c_i64, c_i32, c_p, c_p, c_p, c_p, c_p, c_i32, c_p, c_p],
    "pgg_make_streams": [c_u64, c_i64, c_p, c_p, c_p],
    "pgg_next_u32": [c_i64, c_p, c_p, c_p],
    "pgg_pack_gbuffer": [c_i64] + [c_p] * 15 + [c_p],
    "pgg_pack_gbuffer_mat": [c_i64, c_p, c_p, c_p, c_p, c_p, c_i32, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p,
                             c_p, c_p, c_p],
    "pgg_pack_vpl": [c_i64, c_p, c_p, c_p, c_p, c_p, c_p, c_p],
    "pgg_gamma_split": [c_i64, c_p, c_p, c_p, c_p],
    "pgg_gamma_join": [c_i64, c_p, c_p, c_p, c_p],
    "pgg_gamma_init": [c_i64, c_p, c_p, c_p],
    "pgg_gbuffer_pass": [ctypes.POINTER(Scene), ctypes.POINTER(Camera), ctypes.POINTER(Camera), c_i32, c_i32, c_i32,
                         c_i32, c_p, c_p, c_p, c_p, c_p, c_p, c_p],
    "pgg_render_pass": [ctypes.POINTER(RenderConfig), ctypes.POINTER(Scene), ctypes.POINTER(GBuffer), c_p,
                        ctypes.POINTER(Samples), ctypes.POINTER(RenderOut), c_p],
    "pgg_image_error": [c_i64, c_p, c_p, c_i32, c_p, c_p, c_p],
    "pgg_intersect": [ctypes.POINTER(Scene), c_i64, c_p, c_p, c_p, c_p, c_i32, c_p, c_p, c_p, c_p, c_p, c_p, c_p],
    "pgg_sample_emitter": [ctypes.POINTER(Scene), c_i64, c_p, c_p, c_p, c_p, c_p, c_p, c_p],
    "pgg_brdf": [c_i32, c_i64, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p],
    "pgg_primary_rays": [ctypes.POINTER(Camera), c_i32, c_i32, c_i64, c_p, c_p, c_p, c_p],
    "pgg_sgmap": [c_i32, c_i64, c_p, c_p, c_p],
    "pgg_project": [ctypes.POINTER(Camera), c_i32, c_i32, c_i64, c_p, c_p, c_p, c_p, c_p],
    "pgg_motion_vectors": [ctypes.POINTER(Camera), c_i32, c_i32, c_p, c_p, c_p, c_p, c_p],
    "pgg_mixture_lanes": [c_i32, c_i64, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_i32, c_p],
    "pgg_sample_gauss": [c_i64, c_p, c_p, c_p, c_p, c_p, c_p, c_p],
    "pgg_debug_checks": [c_p, c_i32],
    "pgg_debug_em_offsets": [ctypes.POINTER(Config), c_p, c_p, c_p],
    "pgg_debug_bm_accept": [c_i64, c_i32, c_p, c_p, c_p, c_p, c_p, c_p],
    "pgg_debug_trunc_bvn": [c_i64, c_p, c_p, c_p, c_p],
    "pgg_debug_brdf_draw": [c_i64, c_p, c_p, c_p, c_p, c_p, c_p, c_p],
    "pgg_debug_reproject": [ctypes.POINTER(Config), ctypes.POINTER(GBuffer), ctypes.POINTER(GBuffer),
                            ctypes.POINTER(GammaIn), c_p, c_p],
}

EXPORTS = tuple(_SIGS) + ("pgg_frame_key", "pgg_status_string", "pgg_last_cuda_error", "pgg_abi_version")

_lock = threading.Lock()
_lib = None


def load_library(path=LIB_PATH):
    """dlopen libpgg.so and declare every signature (no device needed)."""
    if not os.path.exists(path):
        raise PggUnavailable(f"{path} not built; run __graft_entry__.build()")
    lib = ctypes.CDLL(path)
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    lib.pgg_frame_key.argtypes = [c_u64, c_u64, c_u64]
    lib.pgg_frame_key.restype = c_u64
    lib.pgg_status_string.argtypes = [ctypes.c_int]
    lib.pgg_status_string.restype = ctypes.c_char_p
    lib.pgg_last_cuda_error.argtypes = []
    lib.pgg_last_cuda_error.restype = ctypes.c_char_p
    lib.pgg_abi_version.argtypes = []
    lib.pgg_abi_version.restype = ctypes.c_int
    return lib


def lib():
    """The loaded library; requires a CUDA device (no CPU path exists)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not torch.cuda.is_available():
                    raise PggUnavailable("no CUDA device: the guiding pass runs only on the GPU (sm_100a)")
                _lib = load_library()
    return _lib


def check(status):
    if status != 0:
        L = lib()
        msg = L.pgg_status_string(status).decode()
        if status == 2:
            msg += ": " + L.pgg_last_cuda_error().decode()
        raise PggError(msg)


def ptr(t):
    """Device pointer of a tensor (None -> NULL)."""
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return ctypes.c_void_p(t.data_ptr())


def stream_ptr(stream=None, device=None):
    """cudaStream_t of ``stream``, default the current stream of ``device``
    (default: the current device)."""
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return ctypes.c_void_p(s.cuda_stream)


def frame_key(seed, frame, stream_id):
    """(seed, frame, stream_id) prefix of rng.make_streams (pg/rng.py:34-36)."""
    return int(lib().pgg_frame_key(int(seed) & 0xFFFFFFFFFFFFFFFF, int(frame) & 0xFFFFFFFFFFFFFFFF,
                                   int(stream_id) & 0xFFFFFFFFFFFFFFFF))
