"""Memory-safety evidence for the fused pass without compute-sanitizer
(closed on this GPU pool): tests/helpers/checked_pass.py runs every
k_guiding_pass instantiation (TMA tile / global VPLs, whole-frame / partial
halo, frame-edge bands, ragged frame sizes, radius 7.3 / 10 / 12 / 13) with
the checked library (libpgg_checked.so: in-kernel bounds asserts on every
shared-memory tile read, global plane read and output store) and with the
product library, and checks sentinel guard rows around every output and
NaN pre-filled outputs: zero bounds failures, every output element written,
no write outside the launch's band.  Race freedom is by construction
 and observed as bitwise determinism
(tests/test_gpu_pass.py, test_gpu_hazards.py::test_concurrent_first_calls)."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
PKG = os.path.join(ROOT, "paper_2112_09728_b200")


@pytest.mark.parametrize("lib", ["libpgg_checked.so", "libpgg.so"])
def test_bounds_and_guards(cuda_dev, lib):
    path = os.path.join(PKG, lib)
    if not os.path.exists(path):
        import __graft_entry__
        __graft_entry__.build()
    env = dict(os.environ, PGG_LIB=path)
    p = subprocess.run([sys.executable, os.path.join("tests", "helpers", "checked_pass.py")], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-4000:]
    rep = json.loads(p.stdout.strip().splitlines()[-1])
    d = os.environ.get("PGG_REPORT_DIR")
    if d:
        os.makedirs(d, exist_ok=True)
        with open(os.path.join(d, f"checked_{lib}.json"), "w") as f:
            json.dump(rep, f, indent=1)
    assert rep["launches"] > 40 and rep["halo_misses"] > 0
    assert rep["unwritten"] == 0 and rep["guard_overwrites"] == 0, rep
    if lib == "libpgg_checked.so":
        assert rep["checked_build"] and rep["check_failures"] == 0, rep
