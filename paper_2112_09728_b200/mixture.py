"""Per-pixel guiding mixture on the GPU; drop-in for pgtrace.mixture
(pg/mixture.py).  Same names, constants, argument meaning and return types.

Every entry point runs a libpgg kernel: lobe_from_stats / truncation_mass
(k_lobe / k_trunc: float64 covariance + reset + Cholesky, exact
bivariate-normal truncation mass), sample_mixture (k_sample_lanes, or
k_sample_gauss + the caller's BRDF callbacks), m_step_update (k_m_step),
gaussian_pdf_square / mixture_pdf / box_muller / e_step_responsibility /
neighbor_count (k_mixture_lanes, float64 in the reference's operation
order).  NumPy inputs return NumPy; CUDA tensors stay on the device.
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
    """Mass of N(mu, cov) inside [0,1]^2, clamped to [1e-4, 1] (pg/mixture.py:84-126).

    The reference's own rule (whitened outer variable, 5 ramp segments x 24
    Gauss-Legendre nodes) in float64 on the device: within 3.5e-13 relative
    of the reference on any input (profiles/r2_trunc_fuzz_*.json).  The fused
    pass evaluates its float32 Genz form instead (7.5e-5 on the lobes it
    forms)."""
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


def _lanes(op, n, a, b=None, c=None, d=None, k_max=0, two=False):
    """Run k_mixture_lanes (float64, reference operation order) on flat device arrays."""
    dev = a.device
    o0 = torch.empty(n, dtype=F64, device=dev)
    o1 = torch.empty(n, dtype=F64, device=dev) if two else None
    _lib.check(_lib.lib().pgg_mixture_lanes(op, n, _lib.ptr(a), _lib.ptr(b), _lib.ptr(c), _lib.ptr(d), None,
                                            _lib.ptr(o0), _lib.ptr(o1), int(k_max), _lib.stream_ptr()))
    return (o0, o1) if two else o0


def _flat(t, lead, tail):
    return t.expand(lead + tail).reshape((-1,) + tail).contiguous()


def gaussian_pdf_square(lobe, p):
    """Truncated-normalised Gaussian density at square points (pg/mixture.py:158-169)."""
    torch_in = _conv.is_torch(p, *lobe)
    L = _lobe_dev(lobe)
    p = _conv.to_dev(p, F64)
    lead = torch.broadcast_shapes(L.mu.shape[:-1], L.chol.shape[:-2], L.trunc_z.shape, p.shape[:-1])
    n = int(np.prod(lead)) if lead else 1
    out = _lanes(0, n, _flat(L.mu, lead, (2,)), _flat(L.chol, lead, (2, 2)), _flat(L.trunc_z, lead, ()),
                 _flat(p, lead, (2,)))
    return _conv.back(out.reshape(lead), torch_in)


def mixture_pdf(stats, lobe, direction, brdf_pdf):
    """pi N(M^-1(dir))/(2 pi) + (1 - pi) brdf_pdf (pg/mixture.py:172-182)."""
    from . import sgmap
    torch_in = _conv.is_torch(stats, direction, brdf_pdf, *lobe)
    st = _conv.to_dev(stats, F64)
    sq = sgmap.hemisphere_to_square(_conv.to_dev(direction, F64))
    L = _lobe_dev(lobe)
    bp = _conv.to_dev(brdf_pdf, F64)
    lead = torch.broadcast_shapes(st.shape[:-1], L.mu.shape[:-1], L.chol.shape[:-2], L.trunc_z.shape,
                                  sq.shape[:-1], bp.shape)
    n = int(np.prod(lead)) if lead else 1
    pk = torch.cat([_flat(L.mu, lead, (2,)), _flat(L.chol, lead, (2, 2)).reshape(n, 4),
                    _flat(L.trunc_z, lead, ()).reshape(n, 1)], dim=1).contiguous()
    out = _lanes(4, n, _flat(st[..., MIX_PI], lead, ()), pk, _flat(sq, lead, (2,)), _flat(bp, lead, ()))
    return _conv.back(out.reshape(lead), torch_in)


def box_muller(u1, u2):
    """Two standard normals; u1 = 0 clamps to 1e-12 (pg/mixture.py:185-190)."""
    torch_in = _conv.is_torch(u1, u2)
    a, b = torch.broadcast_tensors(_conv.to_dev(u1, F64), _conv.to_dev(u2, F64))
    lead = a.shape
    z0, z1 = _lanes(1, a.numel(), a.contiguous().reshape(-1), b.contiguous().reshape(-1), two=True)
    return _conv.back(z0.reshape(lead), torch_in), _conv.back(z1.reshape(lead), torch_in)


def e_step_responsibility(pi, gauss_pdf, brdf_pdf):
    """Posterior of the Gaussian component; 0 where both densities vanish (pg/mixture.py:262-273)."""
    torch_in = _conv.is_torch(pi, gauss_pdf, brdf_pdf)
    a, b, c = torch.broadcast_tensors(*(_conv.to_dev(x, F64) for x in (pi, gauss_pdf, brdf_pdf)))
    lead = a.shape
    out = _lanes(2, a.numel(), *(x.contiguous().reshape(-1) for x in (a, b, c)))
    return _conv.back(out.reshape(lead), torch_in)


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

    Two ways to give the BRDF strategy:

    * the reference's callbacks, exactly as pg/ptrace.py:201-208 passes them:
      ``brdf_sampler(idx, sub_streams) -> (dirs (n,3) local, valid (n,))`` and
      ``brdf_pdf_fn(idx, dirs) -> (n,)``.  The Gaussian branch (zeta draw, up
      to 16 Box-Muller tries) runs on the device (k_sample_gauss); the
      callbacks are then invoked on the host for exactly the lanes and
      stream copies the reference gives them, and the mixture pdf is the
      device's (square map + truncated Gaussian, k_sgmap / k_mixture_lanes).
    * ``mixture.LocalBrdf(kind, roughness, wo_local)`` (brdf_pdf_fn ignored):
      the whole draw, BRDF branch and pdf included, in one kernel
      (k_sample_lanes) -- the fast path _sample_first_bounce uses.

    ``streams`` (uint64, one state per lane) is advanced in place exactly as
    the reference advances it.  Returns (direction (n,3) local, pdf (n,),
    strategy uint8 (n,), valid bool (n,))."""
    if not isinstance(brdf_sampler, LocalBrdf):
        return _sample_mixture_callbacks(stats, lobe, brdf_sampler, brdf_pdf_fn, streams)
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


def _sample_mixture_callbacks(stats, lobe, brdf_sampler, brdf_pdf_fn, streams):
    """sample_mixture with the caller's BRDF callbacks (pg/mixture.py:193-259
    step by step; the callbacks see NumPy arrays, as in the reference)."""
    from . import sgmap
    st = _conv.to_dev(stats, F64).reshape(-1, 8)
    n = st.shape[0]
    L = _lobe_dev(lobe)
    mu = L.mu.reshape(n, 2).contiguous()
    chol = L.chol.reshape(n, 4).contiguous()
    pi = st[:, MIX_PI].contiguous()
    states = _conv.u64_to_dev(streams).reshape(n).clone()
    sq = torch.empty(n, 2, dtype=F64, device=st.device)
    acc = torch.empty(n, dtype=torch.uint8, device=st.device)
    _lib.check(_lib.lib().pgg_sample_gauss(n, _lib.ptr(pi), _lib.ptr(mu), _lib.ptr(chol), _lib.ptr(states),
                                           _lib.ptr(sq), _lib.ptr(acc), _lib.stream_ptr()))
    torch_streams = torch.is_tensor(streams)
    host_streams = streams.cpu().numpy().view(np.uint64) if torch_streams else np.asarray(streams)
    host_streams.reshape(n)[...] = states.cpu().numpy().view(np.uint64)
    accepted = acc.cpu().numpy().astype(bool)
    direction = np.zeros((n, 3))
    if accepted.any():
        direction[accepted] = sgmap.square_to_hemisphere(sq[torch.from_numpy(accepted).to(sq.device)].cpu().numpy())
    brdf_lanes = np.nonzero(~accepted)[0]
    valid = np.ones(n, dtype=bool)
    if brdf_lanes.size:
        hs = host_streams.reshape(n)
        sub = hs[brdf_lanes]
        dirs_b, ok_b = brdf_sampler(brdf_lanes, sub)
        hs[brdf_lanes] = sub
        direction[brdf_lanes] = dirs_b
        valid[brdf_lanes] = ok_b
    if torch_streams:
        streams.view(torch.int64).copy_(torch.from_numpy(host_streams.view(np.int64)).reshape(streams.shape))
    strategy = np.where(accepted, STRATEGY_GAUSSIAN, STRATEGY_BRDF).astype(np.uint8)
    pdf = np.zeros(n)
    ok_idx = np.nonzero(valid)[0]
    if ok_idx.size:
        b = np.asarray(brdf_pdf_fn(ok_idx, direction[ok_idx]), dtype=np.float64)
        sel = torch.from_numpy(ok_idx).to(st.device)
        sub_lobe = GaussianLobe(mu[sel], L.cov.reshape(n, 2, 2)[sel], L.chol.reshape(n, 2, 2)[sel],
                                L.trunc_z.reshape(n)[sel])
        pdf[ok_idx] = mixture_pdf(st[sel], sub_lobe, _conv.to_dev(direction[ok_idx], F64),
                                  _conv.to_dev(b, F64)).cpu().numpy()
    return direction, pdf, strategy, valid


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
    kk = _conv.to_dev(k, F64)
    lead = kk.shape
    out = _lanes(3, kk.numel(), kk.reshape(-1).contiguous(), k_max=int(k_max)).to(torch.int64)
    return _conv.back(out.reshape(lead), torch_in)
