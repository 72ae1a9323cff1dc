"""Wave-quantisation probe: k_guiding_pass time vs frame height at width
1920 (60 tiles per tile-row, 296 resident blocks): a step at whole waves
would show as time / tile-row jumping where 60 R / 296 crosses an integer."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2112_09728_b200 import synth  # noqa: E402
from paper_2112_09728_b200.layout import GBufferPlanes, PassConfig, VplPlanes  # noqa: E402
from paper_2112_09728_b200.session import GuidingSession, run_pass  # noqa: E402

dev = torch.device("cuda:0")
for R in [int(a) for a in sys.argv[1:]] or [74, 79, 84, 86, 88, 89, 90, 92, 94, 98, 99]:
    w, h = 1920, 12 * R
    frames = list(synth.sequence(w, h, 6, seed=0, device=dev))
    cfg = PassConfig(seed=0, spp=1)
    sess = GuidingSession(w, h, cfg, device=dev)
    for f in range(5):
        g, v = frames[f]
        sess.step(GBufferPlanes.from_ref(g, device=dev), VplPlanes.from_ref(v, device=dev), f)
    (gp, _), (gc, vc) = frames[4], frames[5]
    cur, prev, vp = GBufferPlanes.from_ref(gc, device=dev), GBufferPlanes.from_ref(gp, device=dev), VplPlanes.from_ref(vc, device=dev)
    for _ in range(5):
        run_pass(cfg, 5, cur, sess.gamma, prev=prev, vpl=vp)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 50
    e0.record()
    for _ in range(n):
        run_pass(cfg, 5, cur, sess.gamma, prev=prev, vpl=vp)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"R={R} h={h} blocks={60 * R} waves={60 * R / 296:.2f} ms={ms:.4f} ms/tile-row={ms / R * 1000:.3f} us", flush=True)
