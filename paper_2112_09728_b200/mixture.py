"""Per-pixel guiding mixture on the GPU; drop-in for pgtrace.mixture
(pg/mixture.py).  Same names, constants, argument meaning and return types.

Heavy entry points run libpgg kernels: lobe_from_stats / truncation_mass
(k_lobe / k_trunc: float64 covariance + reset + Cholesky, exact
bivariate-normal truncation mass), sample_mixture (k_sample_lanes),
m_step_update (k_m_step).  The remaining one-line densities are float64
elementwise tensor expressions on the same device.  NumPy inputs return
NumPy; CUDA tensors stay on the device.
"""

from typing import NamedTuple

import numpy as np
import torch

from . import _conv, _lib

MEAN_X, MEAN_Y, M2_XX, M2_YY, M2_XY, W_SUM, MIX_PI, EPOCH = range(8)

PI_MIN = 0.05
PI_MAX = 0.95
COV_EPS = 1e-4
EIG_FLOOR = 1e-6
RESET_VAR = 0.05
TRUNC_MIN = 1e-4
KMAX_DEFAULT = 64
MAX_GAUSS_TRIES = 16

STRATEGY_BRDF = 0
STRATEGY_GAUSSIAN = 1

F64 = torch.float64


class GaussianLobe(NamedTuple):
    """mu (...,2), cov (...,2,2), chol (...,2,2) lower, trunc_z (...)
    (pg/mixture.py:34-41)."""

    mu: object
    cov: object
    chol: object
    trunc_z: object


def init_stats(shape=()):
    """Fresh per-pixel state (pg/mixture.py:44-59): centred prior, Sigma =
    0.25 I, pi at its lower clamp, k = 0; float64 NumPy array."""
    shp = tuple(np.atleast_1d(shape)) if shape != () else ()
    row = torch.tensor([0.5, 0.5, 0.5, 0.5, 0.25, 0.0, PI_MIN, 0.0], dtype=F64, device=_conv.device())
    out = row.expand(shp + (8,)).contiguous() if shp else row
    return out.cpu().numpy()


def lobe_from_stats(stats):
    """GaussianLobe from stored moments (pg/mixture.py:129-155)."""
    torch_in = _conv.is_torch(stats)
    st = _conv.to_dev(stats, F64)
    lead = tuple(st.shape[:-1])
    st = st.reshape(-1, 8)
    n = st.shape[0]
    dev = st.device
    mu = torch.empty(n, 2, dtype=F64, device=dev)
    cov = torch.empty(n, 4, dtype=F64, device=dev)
    chol = torch.empty(n, 4, dtype=F64, device=dev)
    z = torch.empty(n, dtype=F64, device=dev)
    _lib.check(_lib.lib().pgg_lobe(n, _lib.ptr(st), _lib.ptr(mu), _lib.ptr(cov), _lib.ptr(chol), _lib.ptr(z), None,
                                   _lib.stream_ptr()))
    return GaussianLobe(_conv.back(mu.reshape(lead + (2,)), torch_in), _conv.back(cov.reshape(lead + (2, 2)), torch_in),
                        _conv.back(chol.reshape(lead + (2, 2)), torch_in), _conv.back(z.reshape(lead), torch_in))


def truncation_mass(mu, cov):
    """Mass of N(mu, cov) inside [0,1]^2, clamped to [1e-4, 1] (pg/mixture.py:84-126)."""
    torch_in = _conv.is_torch(mu, cov)
    m = _conv.to_dev(mu, F64)
    lead = tuple(m.shape[:-1])
    m = m.reshape(-1, 2)
    c = _conv.to_dev(cov, F64).reshape(-1, 4)
    z = torch.empty(m.shape[0], dtype=F64, device=m.device)
    _lib.check(_lib.lib().pgg_trunc_mass(m.shape[0], _lib.ptr(m), _lib.ptr(c), _lib.ptr(z), _lib.stream_ptr()))
    return _conv.back(z.reshape(lead), torch_in)


def _lobe_dev(lobe):
    return GaussianLobe(*[_conv.to_dev(x, F64) for x in lobe])


def gaussian_pdf_square(lobe, p):
    """Truncated-normalised Gaussian density at square points (pg/mixture.py:158-169)."""
    torch_in = _conv.is_torch(p, *lobe)
    L = _lobe_dev(lobe)
    p = _conv.to_dev(p, F64)
    d0 = p[..., 0] - L.mu[..., 0]
    d1 = p[..., 1] - L.mu[..., 1]
    l11, l21, l22 = L.chol[..., 0, 0], L.chol[..., 1, 0], L.chol[..., 1, 1]
    z1 = d0 / l11
    z2 = (d1 - l21 * z1) / l22
    out = torch.exp(-0.5 * (z1 * z1 + z2 * z2)) * (1.0 / (2.0 * np.pi * l11 * l22)) / L.trunc_z
    return _conv.back(out, torch_in)


def mixture_pdf(stats, lobe, direction, brdf_pdf):
    """pi N(M^-1(dir))/(2 pi) + (1 - pi) brdf_pdf (pg/mixture.py:172-182)."""
    from . import sgmap
    torch_in = _conv.is_torch(stats, direction, brdf_pdf, *lobe)
    st = _conv.to_dev(stats, F64)
    sq = sgmap.hemisphere_to_square(_conv.to_dev(direction, F64))
    g = gaussian_pdf_square(_lobe_dev(lobe), sq) / (2.0 * np.pi)
    pi = st[..., MIX_PI]
    out = pi * g + (1.0 - pi) * _conv.to_dev(brdf_pdf, F64)
    return _conv.back(out, torch_in)


def box_muller(u1, u2):
    """Two standard normals; u1 = 0 clamps to 1e-12 (pg/mixture.py:185-190)."""
    torch_in = _conv.is_torch(u1, u2)
    a = torch.clamp(_conv.to_dev(u1, F64), min=1e-12)
    b = _conv.to_dev(u2, F64)
    r = torch.sqrt(-2.0 * torch.log(a))
    ang = 2.0 * np.pi * b
    return _conv.back(r * torch.cos(ang), torch_in), _conv.back(r * torch.sin(ang), torch_in)


class LocalBrdf(NamedTuple):
    """BRDF of the lanes of sample_mixture in their local frame (normal
    e_z): replaces the reference's brdf_sampler / brdf_pdf_fn callbacks,
    which cannot run inside a GPU kernel (pg/ptrace.py:201-208 builds them
    from exactly these three arrays)."""

    kind: object      # (n,) 0 DIFFUSE, 1 GLOSSY
    roughness: object  # (n,)
    wo_local: object   # (n, 3) view direction in the local frame


def _lobe6(lobe):
    L = _lobe_dev(lobe)
    return torch.stack([L.mu[..., 0], L.mu[..., 1], L.chol[..., 0, 0], L.chol[..., 1, 0], L.chol[..., 1, 1],
                        L.trunc_z], dim=-1).to(torch.float32).reshape(-1, 6).contiguous()


def _vec4(v, n):
    v = _conv.to_dev(v, torch.float32).reshape(n, 3)
    return torch.cat([v, torch.zeros(n, 1, dtype=torch.float32, device=v.device)], dim=1).contiguous()


def sample_lanes(world, normal, view, kind, rough, guided, pi, lobe6, states):
    """Run k_sample_lanes; states (n,) int64 device tensor advanced in place."""
    n = states.numel()
    dev = states.device
    direction = torch.empty(n, 4, dtype=torch.float32, device=dev)
    tag = torch.empty(n, dtype=torch.uint8, device=dev)
    glossy = (_conv.to_dev(kind, torch.int32) == 1).to(torch.uint8).reshape(n).contiguous()
    rough = _conv.to_dev(rough, torch.float32).reshape(n).contiguous()
    pi = _conv.to_dev(pi, torch.float32).reshape(n).contiguous()
    nrm = _vec4(normal, n) if world else None
    gd = _conv.to_dev(guided, torch.uint8).reshape(n).contiguous() if world else None
    vw = _vec4(view, n)
    _lib.check(_lib.lib().pgg_sample_lanes(n, 1 if world else 0, _lib.ptr(nrm), _lib.ptr(vw), _lib.ptr(rough),
                                           _lib.ptr(glossy), _lib.ptr(gd), _lib.ptr(pi), _lib.ptr(lobe6),
                                           _lib.ptr(states), _lib.ptr(direction), _lib.ptr(tag), _lib.stream_ptr()))
    return direction, tag


def sample_mixture(stats, lobe, brdf_sampler, brdf_pdf_fn, streams):
    """One-sample mixture draw per lane in the local frame (pg/mixture.py:193-259).

    ``brdf_sampler`` is a LocalBrdf (brdf_pdf_fn is ignored: the pdf of the
    same BRDF is evaluated on the device).  ``streams`` (uint64, one state
    per lane) is advanced in place exactly as the reference advances it.
    Returns (direction (n,3) local, pdf (n,), strategy uint8 (n,), valid bool (n,)).
    """
    if not isinstance(brdf_sampler, LocalBrdf):
        raise TypeError("the GPU sample_mixture takes a mixture.LocalBrdf(kind, roughness, wo_local) in place of "
                        "the reference's Python sampler/pdf callbacks (see INTEGRATION.md)")
    torch_in = _conv.is_torch(stats, streams)
    st = _conv.to_dev(stats, F64).reshape(-1, 8)
    n = st.shape[0]
    states = _conv.u64_to_dev(streams).reshape(n).clone()
    d, t = sample_lanes(False, None, brdf_sampler.wo_local, brdf_sampler.kind, brdf_sampler.roughness, None,
                        st[:, MIX_PI], _lobe6(lobe), states)
    if torch_in:
        streams.view(torch.int64).copy_(states.view(streams.shape))
        return d[:, :3].to(F64), d[:, 3].to(F64), (t & 1), ((t >> 1) & 1).bool()
    np.asarray(streams)[...] = states.cpu().numpy().view(np.uint64).reshape(np.asarray(streams).shape)
    d = d.cpu().numpy().astype(np.float64)
    t = t.cpu().numpy()
    return d[:, :3], d[:, 3], (t & 1).astype(np.uint8), ((t >> 1) & 1).astype(bool)


def e_step_responsibility(pi, gauss_pdf, brdf_pdf):
    """Posterior of the Gaussian component; 0 where both densities vanish (pg/mixture.py:262-273)."""
    torch_in = _conv.is_torch(pi, gauss_pdf, brdf_pdf)
    p = _conv.to_dev(pi, F64)
    g = p * _conv.to_dev(gauss_pdf, F64)
    b = (1.0 - p) * _conv.to_dev(brdf_pdf, F64)
    den = g + b
    out = torch.where(den > 0.0, g / torch.where(den > 0.0, den, torch.ones_like(den)), torch.zeros_like(den))
    return _conv.back(out, torch_in)


def m_step_update(stats, sq, weight, resp, valid=None, k_max=KMAX_DEFAULT):
    """Online weighted M-step (pg/mixture.py:276-321), float64, on the device."""
    torch_in = _conv.is_torch(stats, sq, weight, resp, valid)
    st = _conv.to_dev(stats, F64)
    lead = tuple(st.shape[:-1])
    st = st.reshape(-1, 8)
    n = st.shape[0]
    w = _conv.to_dev(weight, F64)
    c = w.shape[-1] if w.dim() > 0 else 0
    w = w.reshape(n, c)
    r = _conv.to_dev(resp, F64).reshape(n, c)
    q = _conv.to_dev(sq, F64).reshape(n, c, 2)
    v = _conv.to_dev(valid, torch.uint8).reshape(n, c) if valid is not None else None
    out = torch.empty_like(st)
    _lib.check(_lib.lib().pgg_m_step(n, c, _lib.ptr(st), _lib.ptr(q), _lib.ptr(w), _lib.ptr(r), _lib.ptr(v),
                                     int(k_max), _lib.ptr(out), _lib.stream_ptr()))
    return _conv.back(out.reshape(lead + (8,)), torch_in)


def neighbor_count(k, k_max):
    """N = floor((1 - min(k,kMax)/kMax)*15 + 5 + 0.5) (pg/mixture.py:324-328)."""
    torch_in = _conv.is_torch(k)
    kk = torch.clamp(_conv.to_dev(k, F64), max=float(k_max))
    out = torch.floor((1.0 - kk / float(k_max)) * 15.0 + 5.0 + 0.5).to(torch.int64)
    return _conv.back(out, torch_in)
