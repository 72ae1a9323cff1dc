"""Whole-frame parity of the fused pass against the CPU oracle (the tests
check bands and one whole 1080p frame; this checks every pixel and lane of
1080p frames 4 and 12 and of a 4K 4 spp frame).
Usage: python tools/full_frame_parity.py [--json out.json] [--only 1080p|4k]"""
import json
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from helpers.full_frame import run  # noqa: E402

if __name__ == "__main__":
    out = sys.argv[sys.argv.index("--json") + 1] if "--json" in sys.argv else None
    only = sys.argv[sys.argv.index("--only") + 1] if "--only" in sys.argv else None
    recs = []
    if only in (None, "1080p"):
        recs += [run(1920, 1080, 1, 5), run(1920, 1080, 1, 13)]
    if only in (None, "4k"):
        recs.append(run(3840, 2160, 4, 5, chunk=12))
    if out:
        with open(out, "w") as fh:
            json.dump(recs, fh, indent=1)
