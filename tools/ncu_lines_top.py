"""Top source lines of a kernel by executed warp-instructions (and stall
samples) from an ncu source page: ncu -i REP --page source --csv
--print-source cuda,sass > src.csv; python tools/ncu_lines_top.py src.csv [N]"""
import csv
import sys


def main(path, n=60):
    rows = []
    f = None
    tot_i = tot_s = 0
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] == "File Path":
            f = r[1].rsplit("/", 1)[-1]
            continue
        if r[0].isdigit():
            try:
                inst = int(r[7]) if r[7] not in ("-", "") else 0
                st = int(r[4]) if r[4] not in ("-", "") else 0
                thr = float(r[10]) if r[10] not in ("-", "") else 0.0
            except (ValueError, IndexError):
                continue
            tot_i += inst
            tot_s += st
            rows.append((inst, st, thr, f"{f}:{r[0]}", r[1].strip()[:90]))
    rows.sort(reverse=True)
    print(f"total warp-inst {tot_i:.4e} stall samples {tot_s}")
    for inst, st, thr, loc, src in rows[:n]:
        print(f"{100*inst/tot_i:5.2f}% {100*st/max(tot_s,1):5.2f}%st {thr:5.1f}thr {loc:22s} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 60)
