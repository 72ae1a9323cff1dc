"""C ABI: the single-stage entry points equal the fused pass's stages bit for
bit, and the ABI is re-entrant from concurrent host threads on separate
streams (the reference samples from render worker threads)."""

import ctypes
import threading

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _inputs(dev, w=160, h=96, seed=4):
    from paper_2112_09728_b200 import synth
    from paper_2112_09728_b200.layout import GammaPlanes, GBufferPlanes, VplPlanes
    (gp, _), (gc, vc) = list(synth.sequence(w, h, 2, seed=seed, device=dev, first_frame=5))
    cur = GBufferPlanes.from_ref(gc, device=dev)
    prev = GBufferPlanes.from_ref(gp, device=dev)
    vpl = VplPlanes.from_ref(vc, device=dev)
    g = GammaPlanes.fresh(h, w, dev)
    g.g1[..., 3] = torch.randint(0, 40, (h, w), device=dev, dtype=torch.float32)
    g.g0[..., 0] = torch.rand(h, w, device=dev) * 0.5 + 0.25
    return w, h, cur, prev, vpl, g


def test_stage_entry_points_match_fused(cuda_dev):
    from paper_2112_09728_b200 import _lib
    from paper_2112_09728_b200.layout import GammaPlanes, PassConfig, SamplePlanes, make_config
    from paper_2112_09728_b200.session import run_pass
    w, h, cur, prev, vpl, g = _inputs(cuda_dev)
    cfg = PassConfig(seed=3, spp=2)
    fused = run_pass(cfg, 6, cur, g, prev=prev, vpl=vpl, want_reproj=True)
    L = _lib.lib()
    c = make_config(cfg, w, h, 6, prev_cam=prev.cam_origin)
    ca, pa, gi = cur.as_abi(), prev.as_abi(), g.as_in()
    rep = GammaPlanes.empty(h, w, cuda_dev)
    _lib.check(L.pgg_reproject(ctypes.byref(c), ctypes.byref(ca), ctypes.byref(pa), ctypes.byref(gi),
                               ctypes.byref(rep.as_out()), None, _lib.stream_ptr()))
    smp = SamplePlanes.empty(h, w, 2, cuda_dev)
    gri = rep.as_in()
    _lib.check(L.pgg_sample_first_bounce(ctypes.byref(c), ctypes.byref(ca), ctypes.byref(gri),
                                         ctypes.byref(smp.as_abi()), _lib.stream_ptr()))
    tr = GammaPlanes.empty(h, w, cuda_dev)
    va = vpl.as_abi()
    _lib.check(L.pgg_train(ctypes.byref(c), ctypes.byref(ca), ctypes.byref(gri), ctypes.byref(va),
                           ctypes.byref(tr.as_out()), None, _lib.stream_ptr()))
    torch.cuda.synchronize()
    assert torch.equal(rep.g0, fused.gamma_reproj.g0) and torch.equal(rep.g1, fused.gamma_reproj.g1)
    assert torch.equal(smp.dir, fused.samples.dir) and torch.equal(smp.tag, fused.samples.tag)
    assert torch.equal(tr.g0, fused.gamma.g0) and torch.equal(tr.g1, fused.gamma.g1)
    # argument errors: stage outputs required
    assert L.pgg_reproject(ctypes.byref(c), ctypes.byref(ca), None, ctypes.byref(gi), None, None, None) == 1
    assert L.pgg_train(ctypes.byref(c), ctypes.byref(ca), ctypes.byref(gi), None, None, None, None) == 1


def test_concurrent_threads_and_streams(cuda_dev):
    """Four host threads, each on its own CUDA stream, run full passes and
    lane sampling concurrently; every result equals the serial one."""
    from paper_2112_09728_b200.layout import PassConfig
    from paper_2112_09728_b200.session import run_pass
    w, h, cur, prev, vpl, g = _inputs(cuda_dev)
    cfgs = [PassConfig(seed=s, spp=1) for s in range(4)]
    serial = []
    for c in cfgs:
        r = run_pass(c, 6, cur, g, prev=prev, vpl=vpl)
        serial.append((r.gamma.g0.clone(), r.samples.dir.clone()))
    torch.cuda.synchronize()
    out = [None] * 4
    errors = []

    def work(i):
        try:
            s = torch.cuda.Stream(device=cuda_dev)
            with torch.cuda.stream(s):
                for _ in range(5):
                    r = run_pass(cfgs[i], 6, cur, g, prev=prev, vpl=vpl, stream=s)
                s.synchronize()
            out[i] = (r.gamma.g0.clone(), r.samples.dir.clone())
        except Exception as e:  # noqa: BLE001 - reported below
            errors.append(e)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    for i in range(4):
        assert torch.equal(out[i][0], serial[i][0]) and torch.equal(out[i][1], serial[i][1])
    assert not torch.equal(serial[0][1], serial[1][1])  # different seeds really differ
    assert np.isfinite(serial[0][0].cpu().numpy()).all()
