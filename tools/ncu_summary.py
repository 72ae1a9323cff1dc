"""Summarise an ncu report (--set full) of k_guiding_pass into text for
profiles/: headline metrics, stall reasons, and the hottest source lines.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/<name>.txt
    python tools/ncu_summary.py gpurun_out/prof.ncu-rep --traffic 1080p   # -> profiles/traffic.json
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "l1tex__t_bytes.sum",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__cycles_active.avg",
]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


KFILTER = []  # optional ["-k", "regex:<name>"] for multi-kernel reports


def raw_metrics(rep):
    raw = list(csv.reader(io.StringIO(ncu("-i", rep, *KFILTER, "--page", "raw", "--csv"))))
    hdr, vals = raw[0], raw[2] if len(raw) > 2 else raw[1]
    units = raw[1] if len(raw) > 2 else [""] * len(hdr)
    return dict(zip(hdr, vals)), dict(zip(hdr, units))


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit.strip(), 1)
    return float(v.replace(",", "")) * scale


def write_traffic(rep, workload):
    """DRAM read + write bytes of the captured launch -> profiles/traffic.json[workload]."""
    m, u = raw_metrics(rep)
    b = to_bytes(m["dram__bytes_read.sum"], u["dram__bytes_read.sum"]) + \
        to_bytes(m["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
    d = json.load(open(path)) if os.path.exists(path) else {}
    d[workload] = {"dram_bytes_per_launch": b, "warp_instructions_per_launch":
                   float(m["smsp__inst_executed.sum"].replace(",", "")) if "smsp__inst_executed.sum" in m else None,
                   "kernel": m.get("Kernel Name", "?"), "source": os.path.basename(rep)}
    with open(path, "w") as f:
        json.dump(d, f, indent=1)
    print(json.dumps(d[workload]))


def main(rep):
    m, u = raw_metrics(rep)
    print(f"# ncu --set full summary: {rep}")
    print(f"kernel: {m.get('Kernel Name', '?')}")
    print(f"grid {m.get('Grid Size', '?')} block {m.get('Block Size', '?')}")
    for k in KEYS:
        if k in m:
            print(f"{k:62s} {m[k]:>18s} {u.get(k, '')}")
    stalls = {k: v for k, v in m.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_") and
              not k.endswith("_not_issued")}
    tot = sum(float(v) for v in stalls.values() if v.replace(".", "").isdigit()) or 1.0
    print("\n## warp stall samples")
    for k, v in sorted(stalls.items(), key=lambda kv: -float(kv[1]))[:10]:
        print(f"  {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {100 * float(v) / tot:5.1f}%")
    src = list(csv.reader(io.StringIO(ncu("-i", rep, *KFILTER, "--page", "source", "--csv", "--print-source",
                                          "cuda,sass"))))
    cur = hdr2 = None
    agg = []
    for r in src:
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr2 = r
            continue
        if hdr2 and r and r[0].isdigit() and len(r) > 7 and r[2] == "-":
            try:
                agg.append((int(r[4]), int(r[7]), cur, int(r[0]), r[1].strip()[:80]))
            except ValueError:
                pass
    ts = sum(a[0] for a in agg) or 1
    ti = sum(a[1] for a in agg) or 1
    print("\n## hottest source lines (stall samples %, executed warp-instructions %)")
    for a in sorted(agg, reverse=True)[:25]:
        print(f"  {100 * a[0] / ts:5.1f}% {100 * a[1] / ti:5.1f}%  {a[2]}:{a[3]}  {a[4]}")


if __name__ == "__main__":
    if "--kernel" in sys.argv:
        i = sys.argv.index("--kernel")
        KFILTER = ["-k", "regex:" + sys.argv[i + 1]]
        del sys.argv[i:i + 2]
    if len(sys.argv) > 3 and sys.argv[2] == "--traffic":
        write_traffic(sys.argv[1], sys.argv[3])
    else:
        main(sys.argv[1])
