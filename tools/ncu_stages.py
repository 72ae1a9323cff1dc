"""Where the fused pass's instructions go, by stage, from an ncu source page.

usage: ncu -i REP --page source --csv --print-source cuda,sass > src.csv
       python tools/ncu_stages.py src.csv

Each SASS instruction is attributed to the stage of its own source line when
that line is top-level pass code (pgg_pass.cuh / pgg_kernels.cu), else to the
stage of the nearest preceding top-level instruction in address order
(inlined helpers from pgg_math.cuh sit inside their caller's code).  The
stage table below maps pgg_pass.cuh line ranges to the reference functions.
Reports executed warp-instructions, stall samples and mean active lanes per
stage."""
import csv
import re
import sys

# (name, file, first line, last line): anchored on function signatures so
# the ranges follow edits of pgg_pass.cuh
STAGES = [
    ("reproject (guide_buffers.py:78-137)", ["rotate_or_reject", "reproject_px"]),
    ("depth-0 sampling (ptrace.py:161-220, mixture.py:193-259)",
     ["accept_d", "near_edge", "brdf_draw_local_d", "brdf_draw_local", "sample_lane"]),
    ("EM record loop (guide_buffers.py:140-231)",
     ["disk_offset_d", "disk_offset", "pcg_out", "record_valid_d", "em_eval", "em_accumulate", "em_record",
      "em_partial"]),
    ("M-step (mixture.py:276-321)", ["m_step_apply"]),
    ("EM context (lobe constants, BRDF, stream)", ["em_setup"]),
]


def func_ranges(src):
    """first/last line of each named function in pgg_pass.cuh"""
    lines = open(src).read().splitlines()
    starts = []
    for i, l in enumerate(lines, 1):
        m = re.match(r"^(?:template <[^>]*>\s*)?(?:PGG_HD|PGG_COLD|PGG_MHD)\s+[\w:<>,\s&*]+?\b(\w+)\(", l)
        if m:
            starts.append((i, m.group(1)))
    rng = {}
    for k, (i, name) in enumerate(starts):
        end = starts[k + 1][0] - 1 if k + 1 < len(starts) else len(lines)
        rng.setdefault(name, []).append((i, end))
    return rng


def main(path, src="paper_2112_09728_b200/csrc/pgg_pass.cuh"):
    fr = func_ranges(src)
    line_stage = {}
    for stage, funcs in STAGES:
        for f in funcs:
            for a, b in fr.get(f, []):
                for ln in range(a, b + 1):
                    line_stage[ln] = stage
    rows = list(csv.reader(open(path)))
    fname, cur, hdr, data = None, None, None, []
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not hdr or len(r) < 9:
            continue
        if r[2] in ("-", ""):
            cur = (fname, int(r[0]))
            continue
        try:
            data.append((int(r[2], 16), int(r[7]), int(r[4]), int(r[8]), cur))
        except ValueError:
            continue
    data.sort()
    agg = {}
    stage = "kernel prologue / G-buffer loads"
    for a, inst, smp, thr, (f, ln) in data:
        if f == "pgg_pass.cuh":
            if ln in line_stage:
                stage = line_stage[ln]
            elif ln >= fr.get("pixel_stage", [(10 ** 9, 0)])[0][0]:
                stage = "pixel stage: loads, lobe + truncation mass, dispatch"
        elif f == "pgg_kernels.cu":
            stage = "kernel body (TMA, barriers, stores)"
        x = agg.setdefault(stage, [0, 0, 0])
        x[0] += inst
        x[1] += smp
        x[2] += thr
    ti = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    print(f"total warp-instructions {ti}, stall samples {ts}")
    print(f"{'stage':62s} {'inst %':>7s} {'stall %':>8s} {'lanes':>6s}")
    for k, (i, s, t) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{k:62s} {100 * i / ti:7.1f} {100 * s / ts:8.1f} {t / max(i, 1):6.1f}")


if __name__ == "__main__":
    main(*sys.argv[1:])
