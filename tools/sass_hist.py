"""Opcode histogram of one address range of a kernel's SASS.
usage: python tools/sass_hist.py obj_or_so kernel_substring start_hex end_hex [--list]"""
import re
import subprocess
import sys
from collections import Counter

out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
for f in re.split(r"\n\s+Function : ", out):
    if sys.argv[2] not in f.split("\n", 1)[0]:
        continue
    a0, a1 = int(sys.argv[3], 16), int(sys.argv[4], 16)
    body = []
    for l in f.splitlines():
        m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m and a0 <= int(m.group(1), 16) <= a1:
            body.append((m.group(1), m.group(2).strip()))
    ops = Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0].split(".")[0] for _, t in body)
    print(len(body), "instructions")
    for k, v in ops.most_common():
        print(f"{v:5d} {k}")
    if "--list" in sys.argv:
        for a, t in body:
            print(a, t)
    break
