"""The C-ABI library loads without a GPU and exports every symbol that
include/pgg.h declares; the host-side helpers agree with the oracle."""

import os
import re

import numpy as np
import pytest

from oracle import pgg_oracle as O

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2112_09728_b200 import _lib
    return _lib.load_library()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "pgg.h")).read()
    return sorted(set(re.findall(r"\b(pgg_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    names = declared_symbols()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    from paper_2112_09728_b200 import _lib
    assert set(names) == set(_lib.EXPORTS)


def test_abi_version_and_status(lib):
    assert lib.pgg_abi_version() == 2
    assert lib.pgg_status_string(0) == b"ok"
    assert lib.pgg_status_string(1) == b"invalid argument"


@pytest.mark.parametrize("seed,frame,sid", [(0, 0, 0), (3, 1, 1), (123456789, 77, 0), (2**63 + 5, 2**40, 1)])
def test_frame_key_matches_oracle(lib, seed, frame, sid):
    assert lib.pgg_frame_key(seed, frame, sid) == int(O.frame_key(seed, frame, sid))


def test_argument_errors_without_device(lib):
    # argument validation happens before any launch
    assert lib.pgg_lobe(-1, None, None, None, None, None, None, None) == 1
    assert lib.pgg_guiding_pass(None, None, None, None, None, None, None, None, None, None) == 1
    assert lib.pgg_gbuffer_pass(None, None, None, 4, 4, 0, 4, None, None, None, None, None, None, None) == 1
    assert lib.pgg_render_pass(None, None, None, None, None, None, None) == 1


def test_reprojection_refuses_aliased_gamma(lib):
    """With a previous G-buffer the pass reads Gamma at motion-source pixels:
    an output plane shared with the input is refused before any launch (no
    device needed); without reprojection in-place training is allowed past
    this check (it then fails only for lack of a device)."""
    import ctypes
    from paper_2112_09728_b200 import _lib
    cfg = _lib.Config()
    cfg.width, cfg.height, cfg.row0, cfg.rows, cfg.spp, cfg.k_max = 64, 48, 0, 48, 1, 64
    cfg.radius = 10.0
    p = lambda a: ctypes.c_void_p(a)  # noqa: E731  (never dereferenced: refused before launch)
    cur = _lib.GBuffer(p(0x1000), p(0x2000), p(0x3000), p(0x4000), p(0x5000), 0, 48)
    prev = _lib.GBuffer(p(0x6000), p(0x7000), p(0x8000), p(0x9000), p(0xA000), 0, 48)
    gin = _lib.GammaIn(p(0xB000), p(0xC000), 0, 48)
    out_alias = _lib.GammaOut(p(0xC000), p(0xD000))
    out_ok = _lib.GammaOut(p(0xE000), p(0xF000))
    by = ctypes.byref
    assert lib.pgg_guiding_pass(by(cfg), by(cur), by(prev), by(gin), None, None, by(out_alias), None, None,
                                None) == 1
    assert lib.pgg_guiding_pass(by(cfg), by(cur), by(prev), by(gin), None, by(out_alias), None, None, None,
                                None) == 1
    # not refused as an argument error (no CUDA device in this container)
    assert lib.pgg_guiding_pass(by(cfg), by(cur), by(prev), by(gin), None, by(out_ok), None, None, None,
                                None) != 1
    assert lib.pgg_train(by(cfg), by(cur), by(gin), by(_lib.Vpl(p(0x11000), p(0x12000), 0, 48)),
                         by(_lib.GammaOut(p(0xB000), p(0xC000))), None, None) != 1


def test_struct_layout_matches_header():
    import ctypes
    from paper_2112_09728_b200 import _lib
    # pgg_config: 8 int32 + 4 double + double[3] + 2 uint64 = 32 + 32 + 24 + 16
    assert ctypes.sizeof(_lib.Config) == 104
    assert ctypes.sizeof(_lib.GBuffer) == 5 * 8 + 8
    assert ctypes.sizeof(_lib.GammaIn) == 24
    assert ctypes.sizeof(_lib.Vpl) == 24
    # render pass structs
    assert ctypes.sizeof(_lib.Scene) == 8 + 16 + 24
    assert ctypes.sizeof(_lib.Camera) == 13 * 8
    assert ctypes.sizeof(_lib.RenderConfig) == 8 * 4 + 8
    assert ctypes.sizeof(_lib.RenderOut) == 6 * 8


def test_header_constants_match_binding():
    import re
    from paper_2112_09728_b200 import _lib
    src = open(os.path.join(ROOT, "include", "pgg.h")).read()
    assert int(re.search(r"#define PGG_IMAGE_ERROR_SCRATCH (\d+)", src).group(1)) == _lib.IMAGE_ERROR_SCRATCH
    assert int(re.search(r"#define PGG_ABI_VERSION (\d+)", src).group(1)) == 2
