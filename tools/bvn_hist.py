import sys, torch, numpy as np
sys.path.insert(0, ".")
d = torch.load("/tmp/g8.pt")
g = torch.cat([d["g0"], d["g1"]], dim=-1).numpy().reshape(-1, 8).astype(np.float64)
mx, my = g[:, 0], g[:, 1]
sxx = g[:, 2] - mx * mx + 1e-4; syy = g[:, 3] - my * my + 1e-4; sxy = g[:, 4] - mx * my
half = 0.5 * (sxx + syy); dl = np.sqrt(np.maximum(0.25 * (sxx - syy) ** 2 + sxy ** 2, 0))
reset = (half - dl) < 1e-6
sxx[reset] = 0.05; syy[reset] = 0.05; sxy[reset] = 0
r = np.abs(sxy / np.sqrt(sxx * syy))
from scipy.special import ndtr
isx, isy = 1 / np.sqrt(sxx), 1 / np.sqrt(syy)
pa = ndtr((1 - mx) * isx) - ndtr(-mx * isx); pb = ndtr((1 - my) * isy) - ndtr(-my * isy)
need = (sxy != 0) & (np.minimum(1 - pa, 1 - pb) > 1e-6 * pa * pb)
cls = np.select([r < 0.3, r < 0.75, r < 0.925, r < 0.96, r < 0.99, r < 0.999], [4, 6, 10, 12, 16, 24], 0)
cnt = np.where(need & (r < 0.999), cls, 0)
print("reset frac", reset.mean(), "need frac", need.mean())
print("node count hist", {int(k): int(v) for k, v in zip(*np.unique(cnt, return_counts=True))})
w = cnt.reshape(-1, 32)
print("mean nodes/lane", cnt.mean(), "mean warp max", w.max(1).mean(), "sum/32 per warp", (w.sum(1) / 32).mean())
