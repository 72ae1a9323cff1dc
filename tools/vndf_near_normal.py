"""GGX VNDF draws (pgg_debug_brdf_draw) with the view within a small angle
of the normal (|wo.xy| from 1e-7 to 1e-1) against the float64 reference
sampler (pg/scene.py:319-351): max direction error per |wo.xy| decade."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import pgg_oracle as O  # noqa: E402
from paper_2112_09728_b200 import _lib  # noqa: E402

dev = torch.device("cuda:0")
rng = np.random.default_rng(3)
n = 2_000_000
rxy = 10.0 ** rng.uniform(-7, -1, n)
ph = rng.uniform(0, 2 * np.pi, n)
wo = np.stack([rxy * np.cos(ph), rxy * np.sin(ph), np.sqrt(1 - rxy ** 2)], -1).astype(np.float32)
rough = rng.uniform(0.05, 1.0, n).astype(np.float32)
glossy = np.ones(n, np.uint8)
ab = rng.integers(0, 2**32, (n, 2), dtype=np.uint64).astype(np.uint32)
wo4 = np.concatenate([wo, np.zeros((n, 1), np.float32)], axis=1)
out = torch.empty(n, 4, dtype=torch.float32, device=dev)
cnt = torch.zeros(1, dtype=torch.int32, device=dev)
t = lambda a: torch.from_numpy(a).to(dev)  # noqa: E731
g_d, r_d, w_d, ab_d = t(glossy), t(rough), t(wo4), t(ab.view(np.int32))
_lib.check(_lib.lib().pgg_debug_brdf_draw(n, _lib.ptr(g_d), _lib.ptr(r_d), _lib.ptr(w_d), _lib.ptr(ab_d),
                                          _lib.ptr(out), _lib.ptr(cnt), _lib.stream_ptr()))
got = out.cpu().numpy()
u = ab.astype(np.float64) * 2.0 ** -32
alpha = np.maximum(rough.astype(np.float64) ** 2, 1e-6)
d = O._vndf_local(alpha, wo.astype(np.float64), u[:, 0], u[:, 1])
e = np.abs(got[:, :3] - d).max(-1)
dec = np.floor(np.log10(np.hypot(wo[:, 0].astype(np.float64), wo[:, 1])))
for k in range(-7, 0):
    m = dec == k
    if not m.any():
        continue
    print(f"|wo.xy| 1e{k}..1e{k+1}: n={m.sum()} dir err max {e[m].max():.3e} p99.9 {np.percentile(e[m], 99.9):.3e}")
i = int(np.argmax(e))
print("worst", e[i], "wo", wo[i], "rough", rough[i], "u", u[i], "got", got[i], "ref", d[i], "rechecks", int(cnt.item()))
