"""Aggregate an ncu source page (--print-source cuda,sass --csv) by CUDA
source line: stall samples and executed warp instructions per line."""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    cur_file = None
    hdr = None
    agg = []
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and r and r[0].isdigit() and len(r) > 7 and r[2] == "-":
            try:
                samp = int(r[4]); inst = int(r[7])
            except ValueError:
                continue
            agg.append((samp, inst, cur_file, int(r[0]), r[1].strip()[:90]))
    tot_s = sum(a[0] for a in agg) or 1
    tot_i = sum(a[1] for a in agg) or 1
    print(f"total samples {tot_s} warp-inst {tot_i}")
    for a in sorted(agg, reverse=True)[:top]:
        print(f"{100*a[0]/tot_s:5.1f}% smp {100*a[1]/tot_i:5.1f}% inst  {a[2]}:{a[3]}  {a[4]}")
    print("--- by instructions")
    for a in sorted(agg, key=lambda a: -a[1])[:top]:
        print(f"{100*a[0]/tot_s:5.1f}% smp {100*a[1]/tot_i:5.1f}% inst  {a[2]}:{a[3]}  {a[4]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
