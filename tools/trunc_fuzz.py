"""Truncation mass -- the pass's float32 Genz BVN (pgg_debug_trunc_bvn; the
reference rule at |r| >= 0.999) and the API's float64 reference rule
(pgg_trunc_mass) -- against the oracle's restatement of the
reference rule (pg/mixture.py:77-126) on random lobes, with the correlation
concentrated around the node-class boundaries (0.3 / 0.75 / 0.925 / 0.96 /
0.99 / 0.999), means at the square's edges and variances from 1e-7 to 1.
Reports relative error percentiles per |r| class and the worst lobes."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import pgg_oracle as O  # noqa: E402
from paper_2112_09728_b200 import _lib  # noqa: E402

dev = torch.device("cuda:0")
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
n = 2_000_000
edges = np.array([0.3, 0.75, 0.925, 0.96, 0.99, 0.999])
if "--domain" in sys.argv and sys.argv[sys.argv.index("--domain") + 1] == "any":
    rho = rng.uniform(-0.9999, 0.9999, n)
    near = rng.random(n) < 0.4
    rho = np.where(near, rng.choice(edges, n) * rng.choice([-1, 1], n) + rng.normal(0, 2e-4, n), rho)
    rho = np.clip(rho, -0.99999, 0.99999)
    sd = 10.0 ** rng.uniform(-3.5, 0.0, (n, 2))
    mu = rng.uniform(-0.3, 1.3, (n, 2))
    snap = rng.random((n, 2)) < 0.2
    mu = np.where(snap, rng.choice([0.0, 1.0], (n, 2)) + rng.normal(0, 1e-3, (n, 2)), mu)
    sxx, syy = sd[:, 0] ** 2, sd[:, 1] ** 2
    sxy = rho * sd[:, 0] * sd[:, 1]
else:
    # the lobes the pass can form (pg/mixture.py:129-155): means are convex
    # combinations of square points (in [0,1]^2), Sigma = M2 - mu mu^T + 1e-4 I
    # with lambda_min >= 1e-6 (else reset to 0.05 I): eigenvalues 1e-6..0.3
    mu = rng.uniform(0.0, 1.0, (n, 2))
    snap = rng.random((n, 2)) < 0.2
    mu = np.where(snap, np.where(mu < 0.5, rng.uniform(0, 1e-3, (n, 2)), 1.0 - rng.uniform(0, 1e-3, (n, 2))), mu)
    lam = 10.0 ** rng.uniform(-6.0, -0.5, (n, 2))
    th = rng.uniform(0, np.pi, n)
    c, s_ = np.cos(th), np.sin(th)
    sxx = lam[:, 0] * c * c + lam[:, 1] * s_ * s_
    syy = lam[:, 0] * s_ * s_ + lam[:, 1] * c * c
    sxy = (lam[:, 0] - lam[:, 1]) * c * s_
    rho = sxy / np.sqrt(sxx * syy)
    sd = np.stack([np.sqrt(sxx), np.sqrt(syy)], -1)
# the pass sees float32 Gamma: round the moments like it does
cov = np.stack([sxx, sxy, sxy, syy], -1)
mu_d = torch.from_numpy(mu.copy()).to(dev)
cov_d = torch.from_numpy(cov.copy()).to(dev)
z_d = torch.empty(n, dtype=torch.float64, device=dev)
_lib.check(_lib.lib().pgg_debug_trunc_bvn(n, _lib.ptr(mu_d), _lib.ptr(cov_d), _lib.ptr(z_d), _lib.stream_ptr()))
got = z_d.cpu().numpy()
zr_d = torch.empty(n, dtype=torch.float64, device=dev)   # the API: the reference rule in float64
_lib.check(_lib.lib().pgg_trunc_mass(n, _lib.ptr(mu_d), _lib.ptr(cov_d), _lib.ptr(zr_d), _lib.stream_ptr()))
api = zr_d.cpu().numpy()
l11, l21, l22 = O.chol2(sxx, sxy, syy)
ref = np.empty(n)
for a in range(0, n, 1 << 17):
    b = min(n, a + (1 << 17))
    ref[a:b] = O.trunc_mass(mu[a:b, 0], mu[a:b, 1], l11[a:b], l21[a:b], l22[a:b])
rel = np.abs(got - ref) / ref
rel_api = np.abs(api - ref) / ref
cls = np.digitize(np.abs(rho), edges)
out = {"lobes": n, "pass_bvn_rel_p9999": float(np.percentile(rel, 99.99)), "pass_bvn_rel_max": float(rel.max()),
       "api_rel_max": float(rel_api.max()), "per_class": {}}
for c in range(7):
    m = cls == c
    if m.any():
        out["per_class"][f"|r| class {c}"] = {"n": int(m.sum()), "p99.99": float(np.percentile(rel[m], 99.99)),
                                             "max": float(rel[m].max())}
worst = np.argsort(rel)[::-1][:6]
out["worst"] = [dict(rel=float(rel[i]), z=float(ref[i]), got=float(got[i]), mu=mu[i].tolist(), sd=sd[i].tolist(),
                     rho=float(rho[i])) for i in worst]
print(json.dumps(out, indent=1))
