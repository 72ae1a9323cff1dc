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
    _lib.check(_lib.lib().pgg_lobe(n, _lib.ptr(st), _lib.ptr(e(n, 2)), _lib.ptr(e(n, 4)), _lib.ptr(e(n, 4)),
                                   _lib.ptr(e(n)), _lib.ptr(reset), _lib.stream_ptr()))
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


def cpu_sample_rows(threads):
    return 32 * threads


def run_cpu_reference(rows_per_thread=32, threads=None, frame=5, seed=0):
    """Oracle port of the reference path on a bounded sample: `threads`
    row bands of 1920 x rows_per_thread pixels of one 1080p frame, one band
    per host thread (NumPy releases the GIL).  Returns (pixels, seconds, threads)."""
    import numpy as np
    import torch
    from concurrent.futures import ThreadPoolExecutor
    from types import SimpleNamespace

    from oracle import pgg_oracle as O
    from paper_2112_09728_b200 import synth
    threads = threads or (os.cpu_count() or 1)
    h = rows_per_thread * threads
    (gp, _), (gc, vc) = list(synth.sequence(W, h, 2, seed=seed, first_frame=frame - 1))

    def ns(d):
        return SimpleNamespace(**{k: (v.numpy().astype(np.float64) if torch.is_tensor(v) and v.dtype == torch.float32
                                      else (v.numpy() if torch.is_tensor(v) else v)) for k, v in d.items()})

    gpn, gcn, vcn = ns(gp), ns(gc), ns(vc)
    rng = np.random.default_rng(0)
    st = O.fresh_stats(h * W).reshape(h, W, 8).astype(np.float32)
    st[..., 7] = rng.integers(0, 16, (h, W))

    def cut(n, r0, r1):
        return SimpleNamespace(**{k: (v[r0:r1] if isinstance(v, np.ndarray) and v.ndim >= 2 and v.shape[0] == h
                                      else v) for k, v in vars(n).items()})

    stages = {"reproject": 0.0, "sample": 0.0, "train": 0.0}

    def band(i):
        r0, r1 = i * rows_per_thread, (i + 1) * rows_per_thread
        gp_, gc_, vc_ = cut(gpn, r0, r1), cut(gcn, r0, r1), cut(vcn, r0, r1)
        t0 = time.perf_counter()
        g = O.reproject(st[r0:r1], gp_, gc_)           # guide_buffers.reproject
        t1 = time.perf_counter()
        smp = O.sample_frame(g, gc_, seed, frame)        # lobe_from_stats + _sample_first_bounce
        t2 = time.perf_counter()
        tr = O.train(g, vc_, gc_, seed=seed, frame=frame)  # training_pass
        t3 = time.perf_counter()
        if threads == 1:
            stages["reproject"] += t1 - t0
            stages["sample"] += t2 - t1
            stages["train"] += t3 - t2
            # inputs and outputs of the timed sample, for the in-bench parity check
            run_cpu_reference.last_io = dict(gp=gp, gc=gc, vc=vc, gamma_in=st, frame=frame, seed=seed,
                                             gamma_reproj=g, samples=smp, gamma_trained=tr)

    t = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(band, range(threads)))
    if threads == 1:
        run_cpu_reference.last_stages = {k: round(v, 3) for k, v in stages.items()}
    return W * h, time.perf_counter() - t, threads


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
    return {"sample": f"the cpu_baseline input ({got.shape[1]}x{got.shape[0]}, random k in [0, 16))",
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
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    for _ in range(max(args.warmup, 0)):
        run_cpu_reference(rows_per_thread=8, threads=threads)
    px = secs = 0.0
    for _ in range(args.steps):
        p, s, _ = run_cpu_reference(rows_per_thread=8, threads=threads)
        px += p
        secs += s
    mpix = px / secs / 1e6
    sample = f"{threads} row bands of 1920x8 px of a 1080p frame per step (one band per host thread)"
    line = {"impl": "reference", "metric": "guiding-pass Mpixels/s at 1080p", "value": mpix, "unit": "Mpixels/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * secs / args.steps, "ms_per_1080p_frame": 1e3 * W * H / (mpix * 1e6),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "1920x1080 1 spp 16-frame synthetic sequence, fused reproject+sample/pdf(MIS)+EM "
                                   "per frame (BASELINE configs[1]); N>1 = N independent streams",
                       "implementation": "CPU oracle port of pgtrace (reproject, depth-0 sampling, training_pass)",
                       "sample": sample},
            "cpu_baseline": {"value": mpix, "unit": "Mpixels/s", "cores": threads, "kind": "port", "sample": sample},
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
    if world > 1 and not args.no_bands:
        # the strong-scaling leg of the same run: one 4K 4 spp frame over N
        # row bands with the NCCL halo exchange (BASELINE configs[3])
        frames.clear()
        torch.cuda.empty_cache()
        w4, h4, spp4, _ = WORKLOADS["4k4spp"]
        bands = bench_bands(args, rank, world, local_rank, w4, h4, spp4, max(8, min(args.steps, 32)),
                            max(3, args.warmup), "4k4spp")
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        px, secs, thr = run_cpu_reference(rows_per_thread=216, threads=1)
        cpu = {"value": px / secs / 1e6, "unit": "Mpixels/s", "cores": thr, "kind": "port",
               "sample": f"one 1920x216 band of a 1080p frame ({px} px, {secs:.1f} s): reproject + depth-0 "
                         f"sampling + training_pass, oracle port of pgtrace on 1 core",
               "stage_seconds": getattr(run_cpu_reference, "last_stages", None), **cpu_host()}
        cpu["parity"] = parity_vs_cpu(dev)
    if rank == 0:
        metric = ("guiding-pass Mpixels/s at 1080p" if args.workload == "1080p"
                  else f"guiding-pass Mpixels/s ({W}x{H}, {args.spp} spp)")
        line = {"metric": metric, "value": mpix, "unit": "Mpixels/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "ms_per_frame": ms,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic",
                "config": {"workload": "%dx%d %d spp 16-frame synthetic sequence, fused reproject+sample/pdf(MIS)+EM "
                                       "per frame (BASELINE %s); N>1 = N independent streams"
                                       % (W, H, args.spp, WORKLOADS[args.workload][3].split(":")[0]),
                           "l2": "inputs larger than L2 (~200 MB/frame, 16 frames rotating); no flush",
                           "parallelism": "replicas" if world > 1 else "single", **wstats},
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                             "frac": achieved / peak, "traffic": ncu_traffic(args.workload), "peak_kind": peak_kind,
                             "algorithmic_bytes_per_px": bpx, "kernel_ms": kavg,
                             "issue": issue_roofline(args.workload, kavg),
                             "kernel": "k_guiding_pass (fused)"},
                "clocks": clk.summary(),
                "gpu_launches": gpu_launches,
                "e2e": e2e, "cpu_baseline": cpu, "frame_loop": floop}
        if bands is not None:
            line["bands_4k4spp"] = bands
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

    nh = min(4, SEQ)
    host = []
    for i in range(nh):
        g, v = frames[i]
        host.append({k: getattr(g, k).cpu().pin_memory() for k in ("flags", "nd", "pr", "va", "am")} |
                    {"vy": v.y.cpu().pin_memory(), "vl": v.L.cpu().pin_memory(), "cam": g.cam_origin})
    gbs = [GBufferPlanes.empty(H, W, dev) for _ in range(3)]        # cur / prev / next
    vps = [VplPlanes(torch.empty(H, W, 4, device=dev), torch.empty(H, W, 4, device=dev)) for _ in range(2)]
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
            for k in ("flags", "nd", "pr", "va", "am"):
                getattr(cur, k).copy_(hsrc[k], non_blocking=True)
            vp.y.copy_(hsrc["vy"], non_blocking=True)
            vp.L.copy_(hsrc["vl"], non_blocking=True)
            in_done[i % 3].record(s_in)
        cur.cam_origin = hsrc["cam"]
        o = i % 2
        with torch.cuda.stream(s_cmp):
            s_cmp.wait_event(in_done[i % 3])
            if i >= 2:
                s_cmp.wait_event(out_done[o])
            g_in, g_out = gam[st["g"]], gam[1 - st["g"]]
            run_pass(cfg, i % SEQ, cur, g_in, prev=gbs[(i - 1) % 3] if i > 0 else None, vpl=vp, out_gamma=g_out,
                     out_samples=smps[o], stream=s_cmp)
            from paper_2112_09728_b200 import _lib
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
            "path": "pinned host packed planes -> H2D -> pgg_guiding_pass -> pgg_gamma_join + samples -> D2H, "
                    "3 streams (copy-in / pass / copy-out) overlapping adjacent frames"}


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
    use_dist = world > 1 or args.bands
    if use_dist:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    import __graft_entry__
    __graft_entry__.build()
    if args.bands or (world > 1 and args.workload != "1080p"):
        line = bench_bands(args, rank, world, local_rank, W, H, args.spp, args.steps, args.warmup, args.workload)
        if line is not None:
            print(json.dumps(line), flush=True)
    else:
        bench_ours(args, rank, world, local_rank)
    if use_dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
