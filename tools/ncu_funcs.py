"""Executed warp-instructions and mean active lanes per source FUNCTION
(innermost inlined function of each SASS instruction), from an ncu source
page with SASS.  usage: python tools/ncu_funcs.py src.csv [N]"""
import csv
import re
import sys

SRC = {"pgg_math.cuh": "paper_2112_09728_b200/csrc/pgg_math.cuh",
       "pgg_pass.cuh": "paper_2112_09728_b200/csrc/pgg_pass.cuh",
       "pgg_kernels.cu": "paper_2112_09728_b200/csrc/pgg_kernels.cu"}


def starts(path):
    out = []
    for i, l in enumerate(open(path).read().splitlines(), 1):
        m = re.match(r"^\s*(?:template <[^>]*>\s*)?(?:PGG_HD|PGG_COLD|PGG_MHD|PGG_PI|__global__|__device__|int |static )"
                     r"[\w:<>,\s&*]*?\b(\w+)\(", l)
        if m:
            out.append((i, m.group(1)))
    return out


def main(path, n=40):
    fs = {k: starts(v) for k, v in SRC.items()}

    def func(f, line):
        best = "?"
        for i, name in fs.get(f, []):
            if i <= line:
                best = name
        return f"{f}:{best}"

    cur = None
    agg = {}
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] == "File Path":
            cf = r[1].rsplit("/", 1)[-1]
            continue
        if r[0].isdigit():
            cur = func(cf, int(r[0]))
            continue
        if r[0] == "" and r[2].startswith("0x") and cur:
            try:
                inst, thr = int(r[7]), float(r[10])
                st = int(r[4]) if r[4] not in ("", "-") else 0
            except (ValueError, IndexError):
                continue
            a = agg.setdefault(cur, [0, 0.0, 0])
            a[0] += inst
            a[1] += inst * thr
            a[2] += st
    tot = sum(v[0] for v in agg.values())
    tst = sum(v[2] for v in agg.values())
    print(f"total {tot:.4e} warp-inst, {tst} stall samples")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
        print(f"{100 * v[0] / tot:6.2f}% inst {100 * v[2] / max(tst, 1):6.2f}% stall  lanes {v[1] / max(v[0], 1):5.1f}  {k}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
