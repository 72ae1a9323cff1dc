"""List the big loops of a kernel's SASS with their local-memory (LDL/STL) and MUFU counts.
usage: python tools/sass_loops.py obj_or_so kernel_substring"""
import re
import subprocess
import sys

out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
for f in funcs:
    name = f.split("\n", 1)[0]
    if sys.argv[2] not in name:
        continue
    L = [l for l in f.splitlines() if re.search(r"/\*[0-9a-f]{4,}\*/\s+\S", l)]
    addr = lambda l: int(re.search(r"/\*([0-9a-f]{4,})\*/", l).group(1), 16)  # noqa: E731
    print(name[:90], "instructions", len(L), "local ops", sum(1 for x in L if "LDL" in x or "STL" in x))
    for l in L:
        m = re.search(r"BRA (0x[0-9a-f]+)", l)
        if m:
            t, a = int(m.group(1), 16), addr(l)
            if t < a and a - t > 0x600:
                body = [x for x in L if t <= addr(x) <= a]
                print("  loop", hex(t), hex(a), "n", len(body), "local", sum(1 for x in body if "LDL" in x or "STL" in x),
                      "mufu", sum(1 for x in body if "MUFU" in x))
