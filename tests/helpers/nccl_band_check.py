"""Run under torchrun (any N): every rank steps a BandedGuiding with the
NCCL halo exchange (overlapped) on a shared synthetic sequence; rank 0
compares the gathered bands with a whole-frame GuidingSession, bitwise.
Prints 'OK' on success."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))

from paper_2112_09728_b200 import synth  # noqa: E402
from paper_2112_09728_b200.bands import BandedGuiding, gather_rows  # noqa: E402
from paper_2112_09728_b200.layout import GBufferPlanes, PassConfig, VplPlanes  # noqa: E402
from paper_2112_09728_b200.session import GuidingSession  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    W, H, F, seed = 160, 96, 4, 5
    cfg = PassConfig(seed=seed, spp=1)
    band = BandedGuiding(W, H, cfg, rank=rank, world=world, device=dev, max_motion_rows=8)
    whole = GuidingSession(W, H, cfg, device=dev) if rank == 0 else None
    ok = True
    for f, (g, v) in enumerate(synth.sequence(W, H, F, seed=seed, device=dev)):
        full_g, full_v = GBufferPlanes.from_ref(g, device=dev), VplPlanes.from_ref(v, device=dev)
        gb, vp = band.frame_inputs()
        for k in ("flags", "nd", "pr", "va", "am"):
            band.ext_g.own(getattr(gb, k)).copy_(getattr(full_g, k)[band.r0:band.r1])
        gb.cam_origin = full_g.cam_origin
        band.ext_v.own(vp.y).copy_(full_v.y[band.r0:band.r1])
        band.ext_v.own(vp.L).copy_(full_v.L[band.r0:band.r1])
        band.step(f, exchange=True, overlap=True, fallback=True)
        g0, g1 = gather_rows(list(band.gamma_own), rank, world, H)
        if rank == 0:
            whole.step(full_g, full_v, f)
            ok = ok and torch.equal(g0, whole.gamma.g0) and torch.equal(g1, whole.gamma.g1)
    torch.cuda.synchronize()
    if rank == 0:
        print("OK" if ok else "MISMATCH")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
