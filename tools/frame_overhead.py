"""Host-side cost of one RenderSession.run_frame (tiny frame: GPU time ~0)."""
import cProfile
import json
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2112_09728_b200 import cli  # noqa: E402
from paper_2112_09728_b200 import scene as S  # noqa: E402

for mode in ("pg", "pt"):
    sess = cli.RenderSession(S.load_scene("cornell-occluder"), cli.RunConfig(width=8, height=8, mode=mode))
    for f in range(5):
        sess.run_frame(f)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for f in range(5, 105):
        sess.run_frame(f)
    torch.cuda.synchronize()
    print(json.dumps({"mode": mode, "host_ms_per_frame": (time.perf_counter() - t) * 10}))
sess = cli.RenderSession(S.load_scene("cornell-occluder"), cli.RunConfig(width=8, height=8, mode="pg"))
pr = cProfile.Profile()
pr.enable()
for f in range(50):
    sess.run_frame(f)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
