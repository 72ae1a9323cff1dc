"""Fused pass vs a stage-1 / EM-only split (timing probe).  mode fused: the
bench's fused launch; stage1: reproject + samples (no VPLs), writing the
reprojected Gamma; em: the EM launch alone on the reprojected Gamma (run
with PGG_LIB pointing at an EM-only build, -DPGG_PROF_NO_SMP
-DPGG_PROF_NO_REPROJ).  Prints ms per frame over the 16-frame sequence."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2112_09728_b200.layout import GammaPlanes, PassConfig, SamplePlanes  # noqa: E402
from paper_2112_09728_b200.session import run_pass  # noqa: E402

mode = sys.argv[1]
dev = torch.device("cuda:0")
frames = bench.make_frames(dev, 1)
W, H = bench.W, bench.H
cfg = PassConfig(seed=0, spp=1)
g = [GammaPlanes.fresh(H, W, dev), GammaPlanes.empty(H, W, dev), GammaPlanes.empty(H, W, dev)]
smp = SamplePlanes.empty(H, W, 1, dev)
# warm Gamma: 16 fused frames (every mode starts from the same trained state)
st = {"a": 0}
for i in range(16):
    cur, vpl = frames[i % 16]
    r = run_pass(cfg, i, cur, g[st["a"]], prev=frames[(i - 1) % 16][0], vpl=vpl, out_gamma=g[1 - st["a"]],
                 out_samples=smp)
    st["a"] = 1 - st["a"]


def step(i):
    cur, vpl = frames[i % 16]
    prev = frames[(i - 1) % 16][0]
    a = st["a"]
    if mode == "fused":
        run_pass(cfg, i, cur, g[a], prev=prev, vpl=vpl, out_gamma=g[1 - a], out_samples=smp)
    elif mode == "split_sep":  # the split with a separate reprojected-Gamma buffer (not in place)
        run_pass(cfg, i, cur, g[a], prev=prev, vpl=vpl, want_reproj=True, out_reproj=g[2], out_gamma=g[1 - a],
                 out_samples=smp)
    elif mode == "stage1":
        run_pass(cfg, i, cur, g[a], prev=prev, want_reproj=True, out_reproj=g[2], out_samples=smp)
    elif mode == "em":
        run_pass(cfg, i, cur, g[a], vpl=vpl, want_samples=False, out_gamma=g[1 - a])
    st["a"] = 1 - a


for i in range(8):
    step(i)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 96
e0.record()
for i in range(n):
    step(i)
e1.record()
torch.cuda.synchronize()
print(mode, round(e0.elapsed_time(e1) / n, 4), "ms/frame", flush=True)
