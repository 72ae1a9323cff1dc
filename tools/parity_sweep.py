"""Whole-frame parity sweep over seeds and frames (tests/helpers/full_frame):
every pixel and lane against the oracle; prints one summary line per frame
and the worst entries overall.  Usage: python tools/parity_sweep.py [--json out]"""
import json
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from helpers.full_frame import run  # noqa: E402

recs = []
if "--wide" in sys.argv:  # other pass parameters: spp, k_max, radius
    cases = [(1920, 1080, spp, F, seed, kmax, rad) for seed in (11, 12) for F in (3, 9)
             for spp, kmax, rad in ((2, 64, 10.0), (1, 32, 7.3), (4, 16, 12.0))]
else:
    cases = [(1920, 1080, 1, F, seed, 64, 10.0) for seed in (1, 2, 3) for F in (2, 6, 11, 16)]
    cases += [(3840, 2160, 4, 9, 1, 64, 10.0), (1280, 720, 2, 7, 5, 64, 10.0), (2560, 1440, 1, 5, 7, 64, 10.0)]
for w, h, spp, F, seed, kmax, rad in cases:
    r = run(w, h, spp, F, seed=seed, verbose=False, k_max=kmax, radius=rad)
    r["seed"] = seed
    keys = ("gamma_rel_p9999", "gamma_rel_max", "k_mismatches", "strategy_mismatches", "valid_mismatches",
            "dir_abs_max", "pdf_rel_p9999", "pdf_rel_max")
    print(json.dumps({"case": f"{w}x{h} spp{spp} F{F} seed{seed} kmax{kmax} r{rad}", **{k: r[k] for k in keys}}),
          flush=True)
    recs.append(r)
summary = {
    "frames": len(recs),
    "pixels": sum(r["pixels"] for r in recs),
    "lanes": sum(r["lanes"] for r in recs),
    "gamma_rel_max": max(r["gamma_rel_max"] for r in recs),
    "gamma_rel_p9999_max": max(r["gamma_rel_p9999"] for r in recs),
    "k_mismatches": sum(r["k_mismatches"] for r in recs),
    "strategy_mismatches": sum(r["strategy_mismatches"] for r in recs),
    "valid_mismatches": sum(r["valid_mismatches"] for r in recs),
    "dir_abs_max": max(r["dir_abs_max"] for r in recs),
    "pdf_rel_p9999_max": max(r["pdf_rel_p9999"] for r in recs),
    "pdf_rel_max": max(r["pdf_rel_max"] for r in recs),
}
print(json.dumps(summary), flush=True)
if "--json" in sys.argv:
    with open(sys.argv[sys.argv.index("--json") + 1], "w") as fh:
        json.dump({"summary": summary, "frames": recs}, fh, indent=1)
