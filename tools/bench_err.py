"""Time pgg_image_error (mse / rel_mse) on float32 images, L2 flushed between runs."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2112_09728_b200 import _lib
    dev = torch.device("cuda:0")
    out = {}
    big = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    for name, (h, w) in {"1080p": (1080, 1920), "8k": (4320, 7680)}.items():
        a = torch.rand(h, w, 3, device=dev)
        b = torch.rand(h, w, 3, device=dev)
        n = a.numel()
        scratch = torch.empty(_lib.IMAGE_ERROR_SCRATCH, dtype=torch.float64, device=dev)
        res = torch.empty(1, dtype=torch.float64, device=dev)
        for rel in (0, 1):
            ts = []
            for it in range(12):
                big.fill_(it)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                _lib.check(_lib.lib().pgg_image_error(n, _lib.ptr(a), _lib.ptr(b), rel, _lib.ptr(scratch),
                                                      _lib.ptr(res), _lib.stream_ptr()))
                e1.record()
                torch.cuda.synchronize()
                if it >= 2:
                    ts.append(e0.elapsed_time(e1))
            t = sorted(ts)[len(ts) // 2]
            out[f"{name}_rel{rel}"] = {"us": round(t * 1e3, 1), "GB/s": round(8 * n / (t * 1e-3) / 1e9, 1)}
    print(json.dumps({"lib": os.environ.get("PGG_LIB", "default"), **out}))


if __name__ == "__main__":
    main()
