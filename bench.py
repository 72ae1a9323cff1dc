"""Benchmark of the B200 guiding pass (BASELINE.json metric: guiding-pass
ms/frame and Mpixels/s at 1080p; achieved HBM GB/s vs peak).

Workload (BASELINE.json configs[1]): 1920x1080, 1 spp, a 16-frame synthetic
sequence with motion-vector reprojection of Gamma and EM every frame,
cycled.  One step = one fused guiding pass (reproject + lobe + depth-0
guided sampling with MIS pdf + EM over the VPL disk) over one frame, inputs
resident in HBM.  Frame 0 of each cycle carries no history, so Gamma
restarts from init_stats exactly like a fresh RenderSession.  Each frame's
inputs (~200 MB) exceed the 126 MB L2 and 16 frames rotate, so no L2 flush
is needed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1: one rank per GPU under torch.distributed.run (bench.py re-launches
itself that way when started without a torchrun environment; it exits with
an error when fewer than N GPUs are visible or WORLD_SIZE != N).  Every rank
runs its own 1080p stream (8x batched 1080p of configs[4]: replicas, no
collective; "scaling": "weak"; value = N x frames / max-over-ranks time), and
the same line carries "bands_4k4spp": one 4K 4 spp frame split into N row
bands with the overlapped NCCL halo exchange (configs[3], strong scaling).
--impl reference times the CPU reference path (the oracle port of pgtrace,
oracle/pgg_oracle.py) on the host cores, rank 0 only.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

W, H, SEQ = 1920, 1080, 16
WORKLOADS = {  # BASELINE.json configs
    "1080p": (1920, 1080, 1, "configs[1]: 1920x1080 1 spp 16-frame sequence"),
    "4k4spp": (3840, 2160, 4, "configs[3]: 3840x2160 4 spp guiding pass"),
    "8k": (7680, 4320, 1, "configs[4]: 7680x4320 1 spp sequence"),
}
BYTES_PER_PX = 184          # fused pass, 1 spp
BYTES_PER_EXTRA_SPP = 17


METRIC_1080P = "guiding-pass Mpixels/s at 1080p"


def config_1080p(world):
    """The config both arms print (identical dicts: same workload)."""
    return {"workload": "1920x1080 1 spp 16-frame synthetic sequence, fused reproject+sample/pdf(MIS)+EM per frame "
                        "(BASELINE configs[1]); N>1 = N independent streams",
            "parallelism": "replicas" if world > 1 else "single"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=160)
    ap.add_argument("--warmup", type=int, default=16)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--spp", type=int, default=None)
    ap.add_argument("--workload", default="1080p", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-frame-loop", action="store_true")
    ap.add_argument("--bands", action="store_true", help="row-band path even at N=1 (exercises the NCCL code)")
    ap.add_argument("--no-bands", action="store_true", help="N>1: skip the 4K 4 spp row-band leg")
    ap.add_argument("--with-bands-leg", action="store_true",
                    help="run the N>1 row-band leg also at N=1 (under torchrun; exercises that code path)")
    ap.add_argument("--seq", type=int, default=0,
                    help="time one true N-frame sequence (frames generated on the device between passes, "
                         "not timed) instead of cycling 16 resident frames; BASELINE configs[4] is --workload 8k "
                         "--seq 64")
    return ap.parse_args()


def relaunch_under_torchrun(args):
    """`python bench.py --gpus N` (N > 1) without a torchrun environment:
    re-exec this script as N ranks of torch.distributed.run on this node."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def ncu_capture(workload, key):
    """Per-launch figure of k_guiding_pass from the committed `ncu --set full`
    capture (profiles/traffic.json, written by tools/ncu_summary.py
    --traffic): DRAM bytes read + written, or warp instructions issued."""
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(workload, {}).get(key)
    except (OSError, ValueError):
        return None


def ncu_traffic(workload):
    return ncu_capture(workload, "dram_bytes_per_launch")


def issue_roofline(workload, kernel_ms):
    """The bound that actually binds this kernel: warp-instruction issue.
    achieved = ncu's warp instructions per launch / the live kernel time;
    peak = 4 schedulers x SMs x max SM clock (one warp-instruction per
    scheduler per cycle)."""
    inst = ncu_capture(workload, "warp_instructions_per_launch")
    if not inst:
        return None
    import torch
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    mhz = 1965.0
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mhz = float(json.load(f).get("sm_max_mhz", mhz))
    except (OSError, ValueError):
        pass
    achieved = inst / (kernel_ms * 1e-3) / 1e9
    peak = 4 * sms * mhz * 1e6 / 1e9
    return {"achieved": achieved, "peak": peak, "unit": "G warp-inst/s", "frac": achieved / peak,
            "warp_instructions_per_launch": inst}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []      # (host time, fields)
        self.proc = None
        self.window = None  # (t0, t1) of the timed region

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.monotonic(), [c.strip() for c in line.split(",")]))

    def wait_ready(self, timeout=5.0):
        """block until nvidia-smi has produced its first sample (its start-up
        takes longer than a short timed region)"""
        end = time.monotonic() + timeout
        while self.proc and not self.rows and time.monotonic() < end:
            time.sleep(0.01)

    def mark(self, t0, t1):
        self.window = (t0, t1)
        # one sample after the region closes it on both sides
        end = time.monotonic() + 0.5
        while self.proc and not any(t >= t1 for t, _ in self.rows) and time.monotonic() < end:
            time.sleep(0.005)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = [r for _, r in self.rows]
        if self.window:
            # samples inside the timed region (+ one 20 ms sampling period either side)
            t0, t1 = self.window
            inside = [r for t, r in self.rows if t0 - 0.025 <= t <= t1 + 0.025]
            if not inside and self.rows:  # region shorter than the sampling period: nearest samples
                near = sorted(self.rows, key=lambda tr: min(abs(tr[0] - t0), abs(tr[0] - t1)))
                inside = [r for _, r in near[:2]]
            rows = inside or rows[-3:]
        sm = [float(r[0]) for r in rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = set()
        for r in rows:
            for i, n in enumerate(names):
                if len(r) > 3 + i and r[3 + i].lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def make_frames(dev, spp, seed=0):
    """16 frames of packed inputs resident in HBM (generated on the device)."""
    from paper_2112_09728_b200 import synth
    from paper_2112_09728_b200.layout import GBufferPlanes, VplPlanes
    frames = []
    for g, v in synth.sequence(W, H, SEQ, seed=seed, device=dev):
        frames.append((GBufferPlanes.from_ref(g, device=dev), VplPlanes.from_ref(v, device=dev)))
    return frames


def workload_stats(frames, gamma):
    """SURVEY 8(d) reporting: invalid-pixel and history fractions of the
    synthetic frames, and the lobe-reset fraction (lambda_min < 1e-6) of the
    final Gamma over valid pixels (pgg_lobe's reset flags)."""
    import torch

    from paper_2112_09728_b200 import _lib
    fl = torch.stack([g.flags for g, _ in frames])
    valid = (fl & 1).bool()
    hist = ((fl & 3) == 3)
    st = gamma.to_aos().reshape(-1, 8).to(torch.float64).contiguous()
    n = st.shape[0]
    dev = st.device
    e = lambda *s: torch.empty(*s, dtype=torch.float64, device=dev)  # noqa: E731
    reset = torch.empty(n, dtype=torch.uint8, device=dev)
    outs = [e(n, 2), e(n, 4), e(n, 4), e(n)]  # kept alive: a temporary's block could be reused by the next
    _lib.check(_lib.lib().pgg_lobe(n, _lib.ptr(st), *[_lib.ptr(o) for o in outs], _lib.ptr(reset),
                                   _lib.stream_ptr()))
    v_last = valid[(len(frames) - 1)].reshape(-1)
    return {"invalid_fraction": round(1.0 - valid.float().mean().item(), 4),
            "history_fraction": round(hist.float().mean().item() / max(valid.float().mean().item(), 1e-9), 4),
            "reset_fraction": round(reset.bool()[v_last].float().mean().item(), 4)}


def cpu_host():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "host_cores": os.cpu_count()}


def _pgtrace():
    """The unmodified reference package (pip-installed from /root/reference
    into baseline/_ref; it travels to the GPU box with the repo), or None."""
    p = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(p, "pgtrace")) and p not in sys.path:
        sys.path.append(p)
    try:
        from types import SimpleNamespace

        import pgtrace  # noqa: F401
        from pgtrace import guide_buffers, mixture, ptrace, rng
        return SimpleNamespace(gb=guide_buffers, mx=mixture, pt=ptrace, rng=rng)
    except ImportError:
        return None


_FRAMES_1080P = {}


def frame_pair_1080p(frame=5, seed=0):
    """Frames frame-1 and frame of the 1080p bench sequence on the host
    (torch CPU tensors), cached."""
    key = (frame, seed)
    if key not in _FRAMES_1080P:
        from paper_2112_09728_b200 import synth
        _FRAMES_1080P.clear()
        _FRAMES_1080P[key] = list(synth.sequence(1920, 1080, 2, seed=seed, first_frame=frame - 1))
    return _FRAMES_1080P[key]


def band_inputs(r0, r1, frame=5, seed=0):
    """Rows [r0, r1) of the 1080p bench frames as a standalone frame (host
    NumPy; float32 values as the GPU sees them), Gamma = init_stats with k
    drawn in [0, 16) like the first 16 frames of the sequence."""
    import numpy as np
    import torch
    (gp, _), (gc, vc) = frame_pair_1080p(frame, seed)

    def cut(d):
        out = {}
        for k, v in d.items():
            if torch.is_tensor(v) and v.dim() >= 2 and v.shape[0] == 1080:
                out[k] = v[r0:r1].numpy()
            elif k == "height":
                out[k] = r1 - r0
            else:
                out[k] = v.numpy() if torch.is_tensor(v) else v
        return out

    h, w = r1 - r0, 1920
    rng = np.random.default_rng(r0)
    st = np.tile(np.array([0.5, 0.5, 0.5, 0.5, 0.25, 0.0, 0.05, 0.0], np.float32), (h, w, 1))
    st[..., 7] = rng.integers(0, 16, (h, w))
    return dict(gp=cut(gp), gc=cut(gc), vc=cut(vc), gamma_in=st, frame=frame, seed=seed)


def _ref_gbuffer(pg, d):
    import numpy as np
    f64 = lambda k: np.asarray(d[k], np.float64)  # noqa: E731
    h, w = d["valid"].shape
    return pg.pt.GBuffer(width=w, height=h, valid=np.asarray(d["valid"], bool), pos=f64("pos"), normal=f64("normal"),
                         depth=f64("depth"), mat=np.asarray(d["mat"], np.int32), kind=np.asarray(d["kind"], np.int32),
                         albedo=f64("albedo"), roughness=f64("roughness"), front=np.asarray(d["front"], bool),
                         view=f64("view"), motion=f64("motion"), has_history=np.asarray(d["has_history"], bool),
                         cam_origin=np.asarray(d["cam_origin"], np.float64))


def reference_pass(pg, io, spp=1, nee_draws=3, reproject=True):
    """The guiding pass through the reference's OWN functions (pgtrace):
    guide_buffers.reproject (pg/guide_buffers.py:78-137); depth-0 sampling as
    the render issues it (pg/ptrace.py:449-475 lane keys pixel*spp+s, the NEE
    draws, then ptrace._sample_first_bounce, pg/ptrace.py:161-220);
    guide_buffers.training_pass (pg/guide_buffers.py:262-283).  Returns
    (outputs, seconds per stage)."""
    import numpy as np
    from types import SimpleNamespace
    gp, gc = _ref_gbuffer(pg, io["gp"]), _ref_gbuffer(pg, io["gc"])
    h, w = gc.height, gc.width
    v = io["vc"]
    vpl = pg.pt.VplBuffer(np.asarray(v["valid"], bool), np.asarray(v["y"], np.float64),
                          np.asarray(v["radiance"], np.float64), np.asarray(v["strategy"], np.uint8))
    seed, frame = io["seed"], io["frame"]
    t0 = time.perf_counter()
    g = pg.gb.GuidingBuffer(w, h, io["gamma_in"].copy())
    if reproject:
        g = pg.gb.reproject(g, gp, gc, pg.gb.ReprojectionPolicy())
    t1 = time.perf_counter()
    st = g.stats_for_render().reshape(-1, 8)
    valid = gc.valid.reshape(-1)
    idx = np.nonzero(valid)[0]
    lobe = pg.mx.lobe_from_stats(st[idx])
    kind, rough = gc.kind.reshape(-1), gc.roughness.reshape(-1)
    guided = (valid & ((kind == 0) | (rough >= 0.05)) & (st[:, 7] >= 1.0))[idx]
    scene = SimpleNamespace(mat_kind=kind, mat_albedo=gc.albedo.reshape(-1, 3), mat_rough=rough)
    smp = dict(wi=np.zeros((h * w, spp, 3)), pdf=np.zeros((h * w, spp)), strategy=np.zeros((h * w, spp), np.uint8),
               valid=np.zeros((h * w, spp), bool))
    for s_ in range(spp):
        streams = pg.rng.make_streams(seed, frame, np.arange(h * w, dtype=np.uint64) * np.uint64(spp) + np.uint64(s_))
        sub = streams[idx]
        for _ in range(nee_draws):
            pg.rng.next_u32(sub)
        streams[idx] = sub
        wi, pdf, strat, ok = pg.pt._sample_first_bounce(
            scene, idx, gc.pos.reshape(-1, 3)[idx], gc.normal.reshape(-1, 3)[idx], idx, gc.view.reshape(-1, 3)[idx],
            st[idx], lobe, guided, streams)
        smp["wi"][idx, s_], smp["pdf"][idx, s_], smp["strategy"][idx, s_], smp["valid"][idx, s_] = wi, pdf, strat, ok
    t2 = time.perf_counter()
    tr = pg.gb.training_pass(g, vpl, gc, k_max=64, seed=seed, frame_index=frame)
    t3 = time.perf_counter()
    out = dict(gamma_reproj=np.asarray(g.stats), samples=smp, gamma_trained=np.asarray(tr.stats))
    return out, {"reproject": t1 - t0, "sample": t2 - t1, "train": t3 - t2}


def oracle_pass(io, spp=1, reproject=True):
    """The oracle port (oracle/pgg_oracle.py) of the same three stages, used
    only when pgtrace is not importable."""
    import numpy as np
    from types import SimpleNamespace

    from oracle import pgg_oracle as O

    def ns(d):
        return SimpleNamespace(**{k: (np.asarray(v, np.float64) if isinstance(v, np.ndarray) and v.dtype == np.float32
                                      else v) for k, v in d.items()})
    gp, gc, vc = ns(io["gp"]), ns(io["gc"]), ns(io["vc"])
    t0 = time.perf_counter()
    g = O.reproject(io["gamma_in"], gp, gc) if reproject else io["gamma_in"]
    t1 = time.perf_counter()
    smp = O.sample_frame(g, gc, io["seed"], io["frame"], spp=spp)
    t2 = time.perf_counter()
    tr = O.train(g, vc, gc, seed=io["seed"], frame=io["frame"])
    t3 = time.perf_counter()
    return (dict(gamma_reproj=g, samples=smp, gamma_trained=tr),
            {"reproject": t1 - t0, "sample": t2 - t1, "train": t3 - t2})


def run_cpu_reference(rows_per_thread=32, threads=None, frame=5, seed=0):
    """The reference CPU path on a bounded sample of the 1080p workload:
    `threads` row bands of 1920 x rows_per_thread pixels spread evenly over
    frame `frame` of the bench sequence, each run as a standalone frame, one
    band per host thread (NumPy releases the GIL).  pgtrace itself when it
    is importable (kind "reference"), else the oracle port ("port").
    Returns (pixels, seconds, threads, kind)."""
    from concurrent.futures import ThreadPoolExecutor
    threads = threads or (os.cpu_count() or 1)
    pg = _pgtrace()
    kind = "reference" if pg is not None else "port"
    step = 1080 // threads
    bands = [(i * step + (step - rows_per_thread) // 2, i * step + (step - rows_per_thread) // 2 + rows_per_thread)
             for i in range(threads)]
    inputs = [band_inputs(r0, r1, frame, seed) for r0, r1 in bands]

    def band(io):
        return reference_pass(pg, io) if pg is not None else oracle_pass(io)

    t = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        res = list(ex.map(band, inputs))
    secs = time.perf_counter() - t
    if threads == 1:
        run_cpu_reference.last_stages = {k: round(v, 3) for k, v in res[0][1].items()}
        run_cpu_reference.last_io = dict(inputs[0], **res[0][0], rows=bands[0])
    return 1920 * rows_per_thread * threads, secs, threads, kind


def parity_vs_cpu(dev):
    """Run the GPU pass on the exact input the cpu_baseline leg just timed
    (a 1920x216 frame: reproject + 1 spp depth-0 sampling + EM, random k in
    [0, 16)) and compare with the oracle's outputs: SURVEY 8a single-kernel
    policy figures (Gamma per-channel relative error with a 1e-7 floor, k,
    strategy/validity tags, directions, pdfs)."""
    import numpy as np
    import torch

    from paper_2112_09728_b200.layout import GammaPlanes, GBufferPlanes, PassConfig, VplPlanes
    from paper_2112_09728_b200.session import run_pass
    io = getattr(run_cpu_reference, "last_io", None)
    if io is None:
        return None
    cur = GBufferPlanes.from_ref(io["gc"], device=dev)
    prev = GBufferPlanes.from_ref(io["gp"], device=dev)
    r = run_pass(PassConfig(seed=io["seed"], spp=1), io["frame"], cur, GammaPlanes.from_aos(io["gamma_in"], dev),
                 prev=prev, vpl=VplPlanes.from_ref(io["vc"], device=dev), want_reproj=True)
    torch.cuda.synchronize(dev)

    def rel(a, b):
        return np.abs(a.astype(np.float64) - b) / np.maximum(np.abs(b.astype(np.float64)), 1e-7)

    got, ref = r.gamma.to_aos().cpu().numpy(), io["gamma_trained"]
    rep = rel(r.gamma_reproj.to_aos().cpu().numpy(), io["gamma_reproj"])
    g = rel(got, ref)
    n = got.shape[0] * got.shape[1]
    d = r.samples.dir.cpu().numpy().reshape(n, 4)
    t = r.samples.tag.cpu().numpy().reshape(n)
    smp = io["samples"]
    ok = smp["valid"][:, 0] & ((t >> 1) & 1).astype(bool)
    pr = rel(d[ok, 3], smp["pdf"][ok, 0])
    return {"sample": f"the cpu_baseline input: rows {io['rows'][0]}-{io['rows'][1] - 1} of frame {io['frame']} of the "
                      f"1080p sequence as a standalone {got.shape[1]}x{got.shape[0]} frame, k in [0, 16)",
            "against": "pgtrace (the reference itself, baseline/_ref)" if _pgtrace() is not None else "oracle port",
            "gamma_rel_p9999": float(np.percentile(g, 99.99)), "gamma_rel_max": float(g.max()),
            "gamma_reproj_rel_max": float(rep.max()),
            "k_equal": bool(np.array_equal(got[..., 7], ref[..., 7])),
            "tags_equal": bool(np.array_equal(t & 1, smp["strategy"][:, 0]) and
                               np.array_equal(((t >> 1) & 1).astype(bool), smp["valid"][:, 0])),
            "dir_abs_max": float(np.abs(d[:, :3] - smp["wi"][:, 0]).max()),
            "pdf_rel_p9999": float(np.percentile(pr, 99.99)) if pr.size else 0.0,
            "policy": "SURVEY 8a: gamma p99.99 <= 1e-4, max <= 1e-3, k exact; tags exact; dirs <= 1e-5; "
                      "pdf p99.99 <= 1e-4"}


def bench_reference(args, rank, world):
    """--impl reference: the reference's own CPU path (pgtrace from
    baseline/_ref; the oracle port only if it is missing) on all host cores,
    rank 0 only, same metric / unit / config as our arm."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    rows = 8
    kind = "reference"
    for _ in range(max(args.warmup, 0)):
        run_cpu_reference(rows_per_thread=rows, threads=threads)
    px = secs = 0.0
    for _ in range(args.steps):
        p, s_, _, kind = run_cpu_reference(rows_per_thread=rows, threads=threads)
        px += p
        secs += s_
    mpix = px / secs / 1e6
    impl = ("pgtrace (the reference package itself, pip-installed from /root/reference into baseline/_ref): "
            "guide_buffers.reproject, ptrace._sample_first_bounce with the render's lane setup, "
            "guide_buffers.training_pass" if kind == "reference" else "CPU oracle port of pgtrace (oracle/pgg_oracle.py)")
    sample = (f"{threads} row bands of 1920x{rows} px spread over frame 5 of the 1080p sequence, each a standalone "
              f"frame, one band per host thread")
    line = {"impl": "reference", "metric": METRIC_1080P, "value": mpix, "unit": "Mpixels/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * secs / args.steps, "ms_per_1080p_frame": 1e3 * W * H / (mpix * 1e6),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_1080p(world), "implementation": impl, "sample": sample,
            "cpu_baseline": {"value": mpix, "unit": "Mpixels/s", "cores": threads, "kind": kind, "sample": sample,
                             **cpu_host()},
            "e2e": {"value": mpix, "unit": "Mpixels/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def bench_bands(args, rank, world, local_rank, w, h, spp, steps, warmup, workload):
    """configs[3]/[4] at N GPUs: one frame split into N row bands, NCCL halo
    exchange of the EM / reprojection halos every frame, overlapped with the
    band's interior rows (strong scaling).  Returns rank 0's record (None on
    the other ranks)."""
    import torch
    import torch.distributed as dist

    from paper_2112_09728_b200 import synth
    from paper_2112_09728_b200.bands import BandedGuiding
    from paper_2112_09728_b200.layout import GBufferPlanes, PassConfig, VplPlanes

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    cfg = PassConfig(seed=0, spp=spp)
    band = BandedGuiding(w, h, cfg, rank=rank, world=world, device=dev, max_motion_rows=8)
    eg, ev = band.ext_g, band.ext_v
    frames = []
    for g, v in synth.sequence(w, h, SEQ, seed=0, device=dev):
        full_g, full_v = GBufferPlanes.from_ref(g, device=dev), VplPlanes.from_ref(v, device=dev)
        gb, vp = band.extended_planes()
        for name in ("flags", "nd", "pr", "va", "am"):
            eg.own(getattr(gb, name)).copy_(getattr(full_g, name)[band.r0:band.r1])
        gb.cam_origin = full_g.cam_origin
        ev.own(vp.y).copy_(full_v.y[band.r0:band.r1])
        ev.own(vp.L).copy_(full_v.L[band.r0:band.r1])
        frames.append((gb, vp))
        del full_g, full_v
    torch.cuda.synchronize(dev)
    stream = torch.cuda.current_stream(dev)
    state = {"i": 0}

    def step():
        i = state["i"]
        gb, vp = frames[i % SEQ]
        band.step(i % SEQ, gbuf=gb, vpl=vp)
        state["i"] = i + 1

    for _ in range(warmup):
        step()
    torch.cuda.synchronize(dev)
    dist.barrier()
    torch.cuda.synchronize(dev)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        clk.wait_ready()
        h0 = time.monotonic()
        t0.record(stream)
        for _ in range(steps):
            step()
        t1.record(stream)
        torch.cuda.synchronize(dev)
        clk.mark(h0, time.monotonic())
    total = torch.tensor([t0.elapsed_time(t1)], device=dev)
    dist.all_reduce(total, op=dist.ReduceOp.MAX)
    misses = band.halo_misses()
    ms = float(total.item()) / steps
    if rank != 0:
        return None
    peak, peak_kind = peaks()
    bpx = BYTES_PER_PX + BYTES_PER_EXTRA_SPP * (spp - 1)
    achieved = bpx * w * h / (ms * 1e-3) / 1e9 / world
    return {"metric": f"guiding-pass Mpixels/s ({w}x{h}, {spp} spp)", "value": w * h / (ms * 1e-3) / 1e6,
            "unit": "Mpixels/s", "n_gpus": world, "steps": steps, "warmup": warmup, "ms_per_step": ms,
            "ms_per_frame": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOADS[workload][3] + ", row bands + NCCL halo exchange",
                       "parallelism": f"bands{world}",
                       "l2": "inputs larger than L2 (16 frames rotating); no flush"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": ncu_traffic(workload) if world == 1 else None,
                         "peak_kind": peak_kind, "note": "per GPU, step time incl. halo exchange"},
            "clocks": clk.summary(), "gpu_launches": steps * (2 if world > 1 else 1), "halo_misses": misses}


def bench_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2112_09728_b200.layout import GammaPlanes, PassConfig, SamplePlanes
    from paper_2112_09728_b200.session import run_pass

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    cfg = PassConfig(seed=rank, spp=args.spp)
    frames = make_frames(dev, args.spp, seed=rank)
    ga = GammaPlanes.fresh(H, W, dev)
    gb = GammaPlanes.empty(H, W, dev)
    smp = SamplePlanes.empty(H, W, args.spp, dev)
    stream = torch.cuda.current_stream(dev)
    state = {"i": 0, "g": ga, "s": gb}

    def step():
        i = state["i"]
        cur, vpl = frames[i % SEQ]
        prev = frames[(i - 1) % SEQ][0]
        r = run_pass(cfg, i % SEQ, cur, state["g"], prev=prev, vpl=vpl, out_gamma=state["s"], out_samples=smp,
                     stream=stream)
        state["g"], state["s"] = r.gamma, state["g"]
        state["i"] = i + 1

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        clk.wait_ready()
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        h0 = time.monotonic()
        t0.record(stream)
        for k in range(args.steps):
            ev[k][0].record(stream)
            step()
            ev[k][1].record(stream)
        t1.record(stream)
        torch.cuda.synchronize(dev)
        clk.mark(h0, time.monotonic())
        time.sleep(0.05)
    total_ms = t0.elapsed_time(t1)
    kern_ms = [a.elapsed_time(b) for a, b in ev]
    if world > 1:
        tt = torch.tensor([total_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
        dist.barrier()
    ms = total_ms / args.steps
    mpix = world * W * H / (ms * 1e-3) / 1e6
    peak, peak_kind = peaks()
    bpx = BYTES_PER_PX + BYTES_PER_EXTRA_SPP * (args.spp - 1)
    kavg = statistics.mean(kern_ms)
    achieved = bpx * W * H / (kavg * 1e-3) / 1e9

    wstats = workload_stats(frames, state["g"]) if rank == 0 else {}
    gpu_launches = args.steps
    floop = None
    if rank == 0 and world == 1 and args.workload == "1080p" and not args.no_frame_loop:
        floop = bench_frame_loop(dev)
    e2e = None
    if not args.no_e2e:
        e2e = bench_e2e(args, frames, cfg, dev, world)
    bands = None
    if (world > 1 or args.with_bands_leg) and not args.no_bands:
        # the strong-scaling leg of the same run: one 4K 4 spp frame over N
        # row bands with the NCCL halo exchange (BASELINE configs[3])
        frames.clear()
        torch.cuda.empty_cache()
        w4, h4, spp4, _ = WORKLOADS["4k4spp"]
        try:
            bands = bench_bands(args, rank, world, local_rank, w4, h4, spp4, max(8, min(args.steps, 32)),
                                max(3, args.warmup), "4k4spp")
        except Exception as e:  # the headline line must not be lost to the extra leg
            bands = {"error": f"{type(e).__name__}: {e}"[:300]}
            print(f"bench.py: rank {rank}: bands_4k4spp leg failed: {bands['error']}", file=sys.stderr, flush=True)
    cpu = None
    c0 = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.workload == "1080p":
        px, secs, thr, kind = run_cpu_reference(rows_per_thread=216, threads=1)
        cpu = {"value": px / secs / 1e6, "unit": "Mpixels/s", "cores": thr, "kind": kind,
               "sample": f"rows 432-647 of frame 5 of the 1080p sequence as a standalone 1920x216 frame ({px} px, "
                         f"{secs:.1f} s): reproject + depth-0 sampling + training_pass on 1 core, "
                         + ("pgtrace itself (baseline/_ref)" if kind == "reference" else "oracle port of pgtrace"),
               "stage_seconds": getattr(run_cpu_reference, "last_stages", None), **cpu_host()}
        cpu["parity"] = parity_vs_cpu(dev)
        c0 = bench_config0(dev)
    if rank == 0:
        metric = (METRIC_1080P if args.workload == "1080p"
                  else f"guiding-pass Mpixels/s ({W}x{H}, {args.spp} spp)")
        line = {"metric": metric, "value": mpix, "unit": "Mpixels/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "ms_per_frame": ms,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic",
                "config": (config_1080p(world) if args.workload == "1080p" else
                           {"workload": "%dx%d %d spp 16-frame synthetic sequence, fused reproject+sample/pdf(MIS)+EM "
                                        "per frame (BASELINE %s)" % (W, H, args.spp,
                                                                     WORKLOADS[args.workload][3].split(":")[0]),
                            "parallelism": "replicas" if world > 1 else "single"}),
                "l2": "inputs larger than L2 (~200 MB/frame, 16 frames rotating); no flush",
                "workload_stats": wstats,
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                             "frac": achieved / peak, "traffic": ncu_traffic(args.workload), "peak_kind": peak_kind,
                             "algorithmic_bytes_per_px": bpx, "kernel_ms": kavg,
                             "issue": issue_roofline(args.workload, kavg),
                             "kernel": "k_guiding_pass (fused)"},
                "clocks": clk.summary(),
                "gpu_launches": gpu_launches,
                "e2e": e2e, "cpu_baseline": cpu, "frame_loop": floop}
        if c0 is not None:
            line["config0_256"] = c0
        if bands is not None:
            line["bands_4k4spp"] = bands
        print(json.dumps(line), flush=True)


def bench_config0(dev, reps=200):
    """BASELINE configs[0]: a 256x256 synthetic G-buffer + 1 spp radiance
    samples, single-frame EM update and guided sampling -- the GPU pass and
    the reference CPU path (pgtrace, 1 core) on the same frame in the same
    run, with the parity of the two."""
    import numpy as np
    import torch

    from paper_2112_09728_b200 import synth
    from paper_2112_09728_b200.layout import GammaPlanes, GBufferPlanes, PassConfig, VplPlanes
    from paper_2112_09728_b200.session import run_pass
    (gp, _), (gc, vc) = list(synth.sequence(256, 256, 2, seed=0, first_frame=4))
    rng = np.random.default_rng(7)
    st = np.tile(np.array([0.5, 0.5, 0.5, 0.5, 0.25, 0.0, 0.05, 0.0], np.float32), (256, 256, 1))
    st[..., 7] = rng.integers(0, 16, (256, 256))
    npd = lambda d: {k: (v.numpy() if torch.is_tensor(v) else v) for k, v in d.items()}  # noqa: E731
    io = dict(gp=npd(gp), gc=npd(gc), vc=npd(vc), gamma_in=st, frame=5, seed=0)
    cur = GBufferPlanes.from_ref(gc, device=dev)
    vpl = VplPlanes.from_ref(vc, device=dev)
    gin = GammaPlanes.from_aos(st, dev)
    cfg = PassConfig(seed=0, spp=1)
    out = GammaPlanes.empty(256, 256, dev)
    for _ in range(10):
        r = run_pass(cfg, 5, cur, gin, vpl=vpl, out_gamma=out)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        r = run_pass(cfg, 5, cur, gin, vpl=vpl, out_gamma=out, out_samples=r.samples)
    e1.record()
    torch.cuda.synchronize(dev)
    gpu_ms = e0.elapsed_time(e1) / reps
    pg = _pgtrace()
    if pg is not None:
        t = time.perf_counter()
        ref, stages = reference_pass(pg, io, reproject=False)
        cpu_s = time.perf_counter() - t
        kind = "reference"
    else:
        t = time.perf_counter()
        ref, stages = oracle_pass(io, reproject=False)
        cpu_s = time.perf_counter() - t
        kind = "port"
    got = r.gamma.to_aos().cpu().numpy()
    rel = np.abs(got.astype(np.float64) - ref["gamma_trained"]) / np.maximum(np.abs(ref["gamma_trained"]), 1e-7)
    t_ = r.samples.tag.cpu().numpy().reshape(-1)
    d = r.samples.dir.cpu().numpy().reshape(-1, 4)
    return {"workload": "BASELINE configs[0]: 256x256 synthetic G-buffer + 1 spp VPLs, one EM update + guided "
                        "depth-0 sampling (no reprojection), k in [0, 16)",
            "gpu_ms_per_frame": gpu_ms, "gpu_Mpixels_per_s": 65536 / (gpu_ms * 1e-3) / 1e6,
            "gpu_timing": f"CUDA events over {reps} back-to-back launches (inputs 6 MB: L2-resident)",
            "cpu_ms_per_frame": 1e3 * cpu_s, "cpu_Mpixels_per_s": 65536 / cpu_s / 1e6, "cpu_kind": kind,
            "cpu_cores": 1, "cpu_stage_seconds": {k: round(v, 3) for k, v in stages.items()},
            "gpu_vs_cpu": cpu_s * 1e3 / gpu_ms,
            "parity": {"gamma_rel_p9999": float(np.percentile(rel, 99.99)), "gamma_rel_max": float(rel.max()),
                       "k_equal": bool(np.array_equal(got[..., 7], ref["gamma_trained"][..., 7])),
                       "tags_equal": bool(np.array_equal(t_ & 1, ref["samples"]["strategy"][:, 0]) and
                                          np.array_equal(((t_ >> 1) & 1).astype(bool), ref["samples"]["valid"][:, 0])),
                       "dir_abs_max": float(np.abs(d[:, :3] - ref["samples"]["wi"][:, 0]).max())}}


def bench_sequence(args, rank, world, local_rank):
    """BASELINE configs[4]: one true `--seq`-frame sequence (64 at 8K):
    Gamma carried through every frame (k grows to 63, the EM budget shrinks
    from 20 to 5 candidates as in a long run), each frame's inputs generated
    on the device just before its pass (not timed), every pass timed with
    CUDA events on its stream; ms/frame = mean over the sequence, max over
    ranks (N > 1: N independent sequences, weak scaling)."""
    import torch
    import torch.distributed as dist

    from paper_2112_09728_b200 import synth
    from paper_2112_09728_b200.layout import GBufferPlanes, PassConfig, VplPlanes
    from paper_2112_09728_b200.session import GuidingSession
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    sess = GuidingSession(W, H, PassConfig(seed=rank, spp=args.spp), device=dev)
    stream = torch.cuda.current_stream(dev)
    times = []
    with ClockSampler(local_rank) as clk:
        clk.wait_ready()
        h0 = time.monotonic()
        for f, (g, v) in enumerate(synth.sequence(W, H, args.seq, seed=rank, device=dev)):
            gb, vp = GBufferPlanes.from_ref(g, device=dev), VplPlanes.from_ref(v, device=dev)
            del g, v
            torch.cuda.synchronize(dev)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            sess.step(gb, vp, f)
            b.record(stream)
            b.synchronize()
            times.append(a.elapsed_time(b))
        clk.mark(h0, time.monotonic())
    ms = statistics.mean(times)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    if rank != 0:
        return
    peak, peak_kind = peaks()
    bpx = BYTES_PER_PX + BYTES_PER_EXTRA_SPP * (args.spp - 1)
    line = {"metric": f"guiding-pass Mpixels/s ({W}x{H}, {args.spp} spp, {args.seq}-frame sequence)",
            "value": world * W * H / (ms * 1e-3) / 1e6, "unit": "Mpixels/s", "n_gpus": world, "steps": args.seq,
            "warmup": 0, "ms_per_step": ms, "ms_per_frame": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{WORKLOADS[args.workload][3]}, one {args.seq}-frame sequence",
                       "parallelism": "replicas" if world > 1 else "single"},
            "l2": "inputs larger than L2 (one frame is > 3 GB at 8K); no flush",
            "timing": "CUDA events around each fused pass; input generation between passes not timed",
            "ms_first_last_frames": [round(times[0], 4), round(times[-1], 4)],
            "ms_min_max": [round(min(times), 4), round(max(times), 4)],
            "roofline": {"bound": "hbm", "achieved": bpx * W * H / (ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": bpx * W * H / (ms * 1e-3) / 1e9 / peak, "peak_kind": peak_kind,
                         "algorithmic_bytes_per_px": bpx},
            "clocks": clk.summary(), "gpu_launches": args.seq, "e2e": None, "cpu_baseline": None}
    print(json.dumps(line), flush=True)


def bench_frame_loop(dev, frames=16, warmup=4):
    """The whole guided frame on the GPU: G-buffer +
    motion, reproject + depth-0 samples, NEE path lanes writing the VPLs, EM
    (cli.RenderSession on cornell-occluder with a panning camera, 1080p,
    1 spp).  Reported beside the headline; not part of `value`."""
    import torch

    from paper_2112_09728_b200 import cli
    from paper_2112_09728_b200 import scene as S
    doc = S.BUILTIN_SCENES["cornell-occluder"]()
    k0 = dict(doc["camera"][0])
    doc["camera"] = [k0, dict(k0, frame=1000, origin=[k0["origin"][0] + 0.3, k0["origin"][1], k0["origin"][2]])]
    sess = cli.RenderSession(S.scene_from_dict(doc), cli.RunConfig(width=W, height=H, spp=1, mode="pg"),
                             device=dev)
    for f in range(warmup):
        sess.run_frame(f)
    torch.cuda.synchronize(dev)
    per = []
    for f in range(warmup, warmup + frames):  # per-frame events, median (robust to allocator / clock hiccups)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = sess.run_frame(f)
        e1.record()
        torch.cuda.synchronize(dev)
        per.append(e0.elapsed_time(e1))
    ms = statistics.median(per)
    return {"scene": "cornell-occluder (panning)", "ms_per_frame": ms, "Mpixels/s": W * H / (ms * 1e-3) / 1e6,
            "ms_per_frame_min_max": [min(per), max(per)], "mean_path_length": r.mean_path_length,
            "frames": frames, "kernels": "k_gbuffer, k_guiding_pass (reproject+sample), k_render, k_guiding_pass (EM)"}


def bench_e2e(args, frames, cfg, dev, world):
    """Same metric through the public pass API with HOST buffers: every step
    copies its frame's packed inputs pinned-host -> device, runs the fused
    pass, and copies Gamma' (joined to the reference's (H,W,8) layout) and
    the depth-0 samples device -> pinned-host.  Three streams pipeline the
    copies of neighbouring frames under the kernel (copy-in of frame i+1 and
    copy-out of frame i-1 overlap the pass of frame i)."""
    import torch

    from paper_2112_09728_b200.layout import GammaPlanes, GBufferPlanes, SamplePlanes, VplPlanes
    from paper_2112_09728_b200.session import run_pass

    from paper_2112_09728_b200 import _lib, synth
    nh = min(4, SEQ)
    host = []
    # VPLs cross PCIe in the reference's VplBuffer form (valid, y, radiance,
    # strategy: 26 B/px, pg/ptrace.py:67-73) and are packed into the kernel's
    # float4 planes on the device (pgg_pack_vpl); the G-buffer crosses in the
    # packed planes (65 B/px, no padding)
    raw = list(synth.sequence(W, H, nh, seed=cfg.seed, device=dev))
    pin = lambda t, dt: t.to(dt).contiguous().cpu().pin_memory()  # noqa: E731
    f32, u8 = torch.float32, torch.uint8
    for i in range(nh):
        g, v = raw[i]
        # the reference GBuffer's own fields (float32) with its material ids:
        # kind / albedo / roughness come from the scene's material table on
        # the device (pgg_pack_gbuffer_mat, 54 B/px instead of 65 B/px planes)
        host.append({"g_valid": pin(g["valid"], u8), "g_pos": pin(g["pos"], f32), "g_nrm": pin(g["normal"], f32),
                     "g_depth": pin(g["depth"], f32), "g_mat": pin(g["mat"], torch.int32),
                     "g_view": pin(g["view"], f32), "g_motion": pin(g["motion"], f32),
                     "g_hist": pin(g["has_history"], u8),
                     "v_valid": pin(v["valid"], u8), "v_y": pin(v["y"], f32), "v_rad": pin(v["radiance"], f32),
                     "v_strat": pin(v["strategy"], u8), "cam": frames[i][0].cam_origin})
    del raw
    mkind, mrough, malb = (t.contiguous() for t in synth.materials(cfg.seed, dev))
    mkind = mkind.to(torch.int32)
    gkeys = ("g_valid", "g_pos", "g_nrm", "g_depth", "g_mat", "g_view", "g_motion", "g_hist")
    vkeys = ("v_valid", "v_y", "v_rad", "v_strat")
    gbs = [GBufferPlanes.empty(H, W, dev) for _ in range(3)]        # cur / prev / next
    vps = [VplPlanes(torch.empty(H, W, 4, device=dev), torch.empty(H, W, 4, device=dev)) for _ in range(2)]
    vraw = [{k: torch.empty_like(host[0][k], device=dev) for k in gkeys + vkeys} for _ in range(2)]
    # the device packing reproduces the planes the pass benchmark runs on, bit for bit
    chk = vraw[0]
    for k in gkeys:
        chk[k].copy_(host[0][k])
    gchk = GBufferPlanes.empty(H, W, dev)
    _lib.check(_lib.lib().pgg_pack_gbuffer_mat(
        H * W, *[_lib.ptr(chk[k]) for k in gkeys[:5]], int(mkind.numel()), _lib.ptr(mkind), _lib.ptr(malb),
        _lib.ptr(mrough), *[_lib.ptr(chk[k]) for k in gkeys[5:]], _lib.ptr(gchk.flags), _lib.ptr(gchk.nd),
        _lib.ptr(gchk.pr), _lib.ptr(gchk.va), _lib.ptr(gchk.am), _lib.stream_ptr()))
    g0 = frames[0][0]
    if not all(torch.equal(getattr(gchk, k), getattr(g0, k)) for k in ("flags", "nd", "pr", "va", "am")):
        raise RuntimeError("pgg_pack_gbuffer_mat planes differ from the benchmark's G-buffer planes")
    del gchk
    gam = [GammaPlanes.fresh(H, W, dev), GammaPlanes.empty(H, W, dev)]
    smps = [SamplePlanes.empty(H, W, args.spp, dev) for _ in range(2)]
    outs = [torch.empty(H, W, 8, dtype=torch.float32, device=dev) for _ in range(2)]
    h_g = [torch.empty(H, W, 8, dtype=torch.float32).pin_memory() for _ in range(2)]
    h_d = [torch.empty(H, W, args.spp, 4, dtype=torch.float32).pin_memory() for _ in range(2)]
    h_t = [torch.empty(H, W, args.spp, dtype=torch.uint8).pin_memory() for _ in range(2)]
    s_in, s_cmp, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ev = lambda: torch.cuda.Event()  # noqa: E731
    in_done = [ev() for _ in range(3)]
    cmp_done = [ev() for _ in range(3)]
    res_ready = [ev() for _ in range(2)]
    out_done = [ev() for _ in range(2)]
    h2d = sum(t.numel() * t.element_size() for k, t in host[0].items() if k != "cam")
    d2h = h_g[0].numel() * 4 + h_d[0].numel() * 4 + h_t[0].numel()
    st = {"i": 0, "g": 0}

    def step():
        i = st["i"]
        hsrc = host[i % nh]
        cur, vp = gbs[i % 3], vps[i % 2]
        with torch.cuda.stream(s_in):
            if i >= 2:
                s_in.wait_event(cmp_done[(i - 2) % 3])    # slot last read by pass i-1 (as prev) / i-2
            for k, t in vraw[i % 2].items():
                t.copy_(hsrc[k], non_blocking=True)
            in_done[i % 3].record(s_in)
        cur.cam_origin = hsrc["cam"]
        o = i % 2
        with torch.cuda.stream(s_cmp):
            s_cmp.wait_event(in_done[i % 3])
            if i >= 2:
                s_cmp.wait_event(out_done[o])
            g_in, g_out = gam[st["g"]], gam[1 - st["g"]]
            r = vraw[i % 2]
            _lib.check(_lib.lib().pgg_pack_gbuffer_mat(
                H * W, *[_lib.ptr(r[k]) for k in gkeys[:5]], int(mkind.numel()), _lib.ptr(mkind), _lib.ptr(malb),
                _lib.ptr(mrough), *[_lib.ptr(r[k]) for k in gkeys[5:]], _lib.ptr(cur.flags), _lib.ptr(cur.nd),
                _lib.ptr(cur.pr), _lib.ptr(cur.va), _lib.ptr(cur.am), _lib.stream_ptr(s_cmp)))
            _lib.check(_lib.lib().pgg_pack_vpl(H * W, _lib.ptr(r["v_valid"]), _lib.ptr(r["v_y"]),
                                               _lib.ptr(r["v_rad"]), _lib.ptr(r["v_strat"]), _lib.ptr(vp.y),
                                               _lib.ptr(vp.L), _lib.stream_ptr(s_cmp)))
            run_pass(cfg, i % SEQ, cur, g_in, prev=gbs[(i - 1) % 3] if i > 0 else None, vpl=vp, out_gamma=g_out,
                     out_samples=smps[o], stream=s_cmp)
            _lib.check(_lib.lib().pgg_gamma_join(H * W, _lib.ptr(g_out.g0), _lib.ptr(g_out.g1), _lib.ptr(outs[o]),
                                                 _lib.stream_ptr(s_cmp)))
            cmp_done[i % 3].record(s_cmp)
            res_ready[o].record(s_cmp)
        st["g"] = 1 - st["g"]
        with torch.cuda.stream(s_out):
            s_out.wait_event(res_ready[o])
            h_g[o].copy_(outs[o], non_blocking=True)
            h_d[o].copy_(smps[o].dir, non_blocking=True)
            h_t[o].copy_(smps[o].tag, non_blocking=True)
            out_done[o].record(s_out)
        st["i"] = i + 1

    steps = max(4, min(args.steps, 32))
    for _ in range(3):
        step()
    torch.cuda.synchronize(dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s_in)
    for _ in range(steps):
        step()
    s_out.wait_stream(s_cmp)
    b.record(s_out)
    torch.cuda.synchronize(dev)
    ms = a.elapsed_time(b) / steps
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return {"value": world * W * H / (ms * 1e-3) / 1e6, "unit": "Mpixels/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": ms, "steps": steps,
            "path": "pinned host: the reference's GBuffer fields (float32, material ids) + VplBuffer fields -> "
                    "H2D -> pgg_pack_gbuffer_mat + pgg_pack_vpl -> pgg_guiding_pass -> pgg_gamma_join + samples -> "
                    "D2H, 3 streams (copy-in / pass / copy-out) overlapping adjacent frames"}


def main():
    global W, H
    args = parse()
    W, H, spp0, _ = WORKLOADS[args.workload]
    if args.spp is None:
        args.spp = spp0
    if args.gpus < 1:
        sys.exit(f"bench.py: --gpus must be >= 1 (got {args.gpus})")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        if args.impl != "reference":
            import torch
            n = torch.cuda.device_count()
            if n < args.gpus:
                sys.exit(f"bench.py: --gpus {args.gpus} requested but only {n} CUDA device(s) are visible")
        relaunch_under_torchrun(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        sys.exit(f"bench.py: rank {rank}: WORLD_SIZE={world} but --gpus {args.gpus}")
    if args.impl == "reference":
        bench_reference(args, rank, world)
        return
    import torch
    import torch.distributed as dist
    if torch.cuda.device_count() <= local_rank:
        sys.exit(f"bench.py: rank {rank}: LOCAL_RANK={local_rank} but only {torch.cuda.device_count()} "
                 "CUDA device(s) are visible")
    use_dist = world > 1 or args.bands or args.with_bands_leg
    if use_dist:
        if "RANK" not in os.environ:  # one process without torchrun: a world of one
            import socket
            with socket.socket() as so:
                so.bind(("127.0.0.1", 0))
                port = so.getsockname()[1]
            os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                              MASTER_PORT=str(port))
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    import __graft_entry__
    if use_dist and world > 1:
        # one compile per node: the other ranks wait, then find it up to date
        if local_rank == 0:
            __graft_entry__.build()
        dist.barrier()
        if local_rank != 0:
            __graft_entry__.build()
    else:
        __graft_entry__.build()
    if args.seq:
        bench_sequence(args, rank, world, local_rank)
    elif args.bands or (world > 1 and args.workload != "1080p"):
        line = bench_bands(args, rank, world, local_rank, W, H, args.spp, args.steps, args.warmup, args.workload)
        if line is not None:
            print(json.dumps(line), flush=True)
    else:
        bench_ours(args, rank, world, local_rank)
    if use_dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
