"""Per source line: executed warp-instructions and mean active lanes, from
an ncu source page with SASS (ncu -i REP --page source --csv --print-source
cuda,sass).  SASS rows are attributed to the source line heading them.
usage: python tools/ncu_lines_lanes.py src.csv FILE LINE_FROM LINE_TO"""
import csv
import sys


def main(path, fname, lo, hi):
    cur_file, cur_line = None, None
    agg = {}
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].rsplit("/", 1)[-1]
            continue
        if r[0].isdigit():
            cur_line = (cur_file, int(r[0]), r[1].strip()[:70])
            continue
        if r[0] == "" and r[2].startswith("0x") and cur_line:
            try:
                inst = int(r[7])
                thr = float(r[10])
            except (ValueError, IndexError):
                continue
            a = agg.setdefault(cur_line, [0, 0.0])
            a[0] += inst
            a[1] += inst * thr
    tot = sum(v[0] for v in agg.values())
    sel = [(k, v) for k, v in agg.items() if k[0] == fname and lo <= k[1] <= hi]
    s_inst = sum(v[0] for _, v in sel)
    s_thr = sum(v[1] for _, v in sel)
    print(f"{fname}:{lo}-{hi}: {100 * s_inst / tot:.2f}% of warp-inst, mean lanes {s_thr / max(s_inst, 1):.1f}")
    for k, v in sorted(sel, key=lambda kv: kv[0][1]):
        if v[0]:
            print(f"  {k[1]:5d} {100 * v[0] / tot:6.3f}%  lanes {v[1] / v[0]:5.1f}  {k[2]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))
