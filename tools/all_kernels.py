"""Launch every libpgg kernel once or twice at 1080p-sized inputs through the
public APIs, for one ncu pass that records each kernel's DRAM bytes and
duration (tools/all_kernels.sh -> profiles/r1_all_kernels_hbm.txt).  Not a
benchmark: the numbers that matter come from ncu, not from this process."""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

W, H = 1920, 1080
N = W * H


def main():
    from paper_2112_09728_b200 import cli, metrics, mixture, rng, scene, sgmap, synth
    from paper_2112_09728_b200.layout import GammaPlanes, GBufferPlanes, PassConfig, SamplePlanes, VplPlanes
    from paper_2112_09728_b200.session import run_pass
    dev = torch.device("cuda:0")
    r = np.random.default_rng(0)
    steps = []

    def step(name, fn):
        steps.append((name, fn))

    (gp, _), (gc, vc) = list(synth.sequence(W, H, 2, seed=1, device=dev, first_frame=3))
    cur = GBufferPlanes.from_ref(gc, device=dev)       # k_pack_gbuffer
    prev = GBufferPlanes.from_ref(gp, device=dev)
    vpl = VplPlanes.from_ref(vc, device=dev)           # k_pack_vpl
    g_in = GammaPlanes.fresh(H, W, dev)                # k_gamma_init
    g_out = GammaPlanes.empty(H, W, dev)
    smp = SamplePlanes.empty(H, W, 1, dev)
    cfg = PassConfig()
    step("k_guiding_pass (tile)", lambda: run_pass(cfg, 3, cur, g_in, prev=prev, vpl=vpl, out_gamma=g_out,
                                                   out_samples=smp))
    aos = g_out.to_aos()                                # k_gamma_join
    step("k_gamma_join", lambda: g_out.to_aos())
    step("k_gamma_split", lambda: GammaPlanes.from_aos(aos, device=dev))

    n = 1 << 20
    stats = np.tile(mixture.init_stats(), (n, 1))
    stats[:, 0:2] = r.uniform(0.2, 0.8, (n, 2))
    stats[:, 2:4] = stats[:, 0:2] ** 2 + r.uniform(0.001, 0.05, (n, 2))
    stats[:, 4] = stats[:, 0] * stats[:, 1] + r.uniform(-0.005, 0.005, n)
    stats[:, 7] = r.integers(0, 64, n)
    step("k_lobe", lambda: mixture.lobe_from_stats(stats))
    lb = mixture.lobe_from_stats(stats)
    step("k_trunc", lambda: mixture.truncation_mass(lb.mu, lb.cov))
    m = 1 << 18
    sq = r.uniform(0, 1, (m, 20, 2))
    w = r.exponential(1.0, (m, 20))
    resp = r.uniform(0, 1, (m, 20))
    step("k_m_step", lambda: mixture.m_step_update(stats[:m], sq, w, resp, k_max=64))
    lanes = np.arange(n, dtype=np.uint64)
    step("k_make_streams", lambda: rng.make_streams(1, 2, lanes))
    st = rng.make_streams(1, 2, lanes)
    step("k_next_u32", lambda: rng.next_u32(st))
    pts = r.uniform(0, 1, (n, 2))
    step("k_lane_sgmap (square_to_hemisphere)", lambda: sgmap.square_to_hemisphere(pts))

    sc = scene.load_scene("cornell-occluder")
    sess = cli.RenderSession(sc, cli.RunConfig(width=W, height=H, spp=1, mode="pg"), device=dev)
    step("frame loop (k_gbuffer, k_guiding_pass, k_render)", lambda: sess.run_frame(len(steps)))
    img_a = torch.rand(H, W, 3, device=dev)
    img_b = torch.rand(H, W, 3, device=dev)
    step("k_err_partial / k_err_final", lambda: metrics.rel_mse(img_a, img_b))
    o = torch.from_numpy(r.uniform(-0.5, 0.5, (n, 3))).to(dev)
    d = torch.nn.functional.normalize(torch.from_numpy(r.normal(size=(n, 3))).to(dev), dim=1)
    step("k_lane_intersect", lambda: scene.intersect(sc, o, d))

    for name, fn in steps:
        for _ in range(2):
            fn()
        torch.cuda.synchronize(dev)
        print("ok", name, flush=True)


if __name__ == "__main__":
    main()
