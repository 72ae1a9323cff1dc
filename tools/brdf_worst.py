"""Worst direction errors of the sampler's BRDF draws vs the float64
reference (same inputs as tests/test_gpu_hazards.py::test_brdf_draws_10m)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import pgg_oracle as O  # noqa: E402
from paper_2112_09728_b200 import _lib  # noqa: E402

dev = torch.device("cuda:0")
rng = np.random.default_rng(17)
n = 10_500_000
glossy = (rng.random(n) < 2 / 3).astype(np.uint8)
rough = rng.uniform(0.05, 1.0, n).astype(np.float32)
rough[rng.random(n) < 0.1] = np.float32(0.05)
wo = rng.normal(size=(n, 3))
wo[:, 2] = np.abs(wo[:, 2]) * np.where(rng.random(n) < 0.2, 0.02, 1.0)
wo[rng.random(n) < 0.01, 2] *= -1.0
wo /= np.linalg.norm(wo, axis=1, keepdims=True)
wo = wo.astype(np.float32)
ab = rng.integers(0, 2**32, (n, 2), dtype=np.uint64).astype(np.uint32)
wo4 = np.concatenate([wo, np.zeros((n, 1), np.float32)], axis=1)
out = torch.empty(n, 4, dtype=torch.float32, device=dev)
cnt = torch.zeros(1, dtype=torch.int32, device=dev)
keep = [torch.from_numpy(a).to(dev) for a in (glossy, rough, wo4, ab.view(np.int32))]  # alive until the launch ran
_lib.check(_lib.lib().pgg_debug_brdf_draw(n, *[_lib.ptr(k) for k in keep], _lib.ptr(out), _lib.ptr(cnt),
                                          _lib.stream_ptr()))
torch.cuda.synchronize()
got = out.cpu().numpy()
u = ab.astype(np.float64) * 2.0 ** -32
wl = wo.astype(np.float64)
alpha = np.maximum(rough.astype(np.float64) ** 2, 1e-6)
gl = glossy.astype(bool)
d = O._cosine_local(u[:, 0], u[:, 1])
d[gl] = O._vndf_local(alpha[gl], wl[gl], u[gl, 0], u[gl, 1])
ok = (d[:, 2] > 1e-9) & (wl[:, 2] > 0.0)
err = np.where(ok, np.abs(got[:, :3] - d).max(1), 0)
idx = np.argsort(-err)[:12]
print("rechecks", int(cnt.item()), "n>1e-5", int((err > 1e-5).sum()), "n>5e-6", int((err > 5e-6).sum()))
for i in idx:
    print(i, "err %.3e" % err[i], "glossy", glossy[i], "alpha %.4g" % alpha[i], "wo", wo[i], "u", u[i], "ref", d[i], "got",
          got[i, :3])
