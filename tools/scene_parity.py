"""Whole-frame parity of the fused pass on rendered inputs at 1080p for the
three built-in scenes (tests/helpers/scene_frame.py; the GPU suite runs two
of them at 640x360).  Usage: python tools/scene_parity.py [F] [--json out.json]"""
import json
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from helpers.scene_frame import one  # noqa: E402

if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    out = sys.argv[sys.argv.index("--json") + 1] if "--json" in sys.argv else None
    if out in args:
        args.remove(out)
    F = int(args[0]) if args else 6
    recs = [one(n, F) for n in ("cornell-occluder", "glossy-box", "indirect-corridor")]
    if out:
        with open(out, "w") as fh:
            json.dump(recs, fh, indent=1)
