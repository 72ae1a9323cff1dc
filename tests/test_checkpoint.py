"""PGG1 checkpoint IO (pg/guide_buffers.py:289-314; SPEC.md section on
checkpoints): host-side file format, no GPU needed."""

import struct

import numpy as np
import pytest

from paper_2112_09728_b200 import guide_buffers as GB


def test_roundtrip_and_format(tmp_path):
    st = np.random.default_rng(0).uniform(0, 1, (9, 17, 8)).astype(np.float32)
    p = tmp_path / "g.pgg"
    GB.checkpoint_save(GB.GuidingBuffer(17, 9, st), p)
    raw = p.read_bytes()
    assert raw[:4] == b"PGG1" and struct.unpack("<II", raw[4:12]) == (17, 9)
    assert len(raw) == 12 + 17 * 9 * 8 * 4
    g = GB.checkpoint_load(p, expect_size=(17, 9))
    np.testing.assert_array_equal(g.stats, st)
    assert (g.width, g.height) == (17, 9)


def test_errors(tmp_path):
    p = tmp_path / "bad.pgg"
    p.write_bytes(b"PGG0" + struct.pack("<II", 1, 1) + b"\0" * 32)
    with pytest.raises(GB.CheckpointError, match="magic"):
        GB.checkpoint_load(p)
    p.write_bytes(b"PGG1" + b"\1\0")
    with pytest.raises(GB.CheckpointError, match="header"):
        GB.checkpoint_load(p)
    p.write_bytes(b"PGG1" + struct.pack("<II", 2, 2) + b"\0" * 10)
    with pytest.raises(GB.CheckpointError, match="payload"):
        GB.checkpoint_load(p)
    p.write_bytes(b"PGG1" + struct.pack("<II", 64, 64) + b"\0" * (64 * 64 * 32))
    with pytest.raises(GB.CheckpointError, match="64x64"):
        GB.checkpoint_load(p, expect_size=(32, 32))


def test_reference_file_compat(tmp_path):
    """A file written the reference's way loads here and vice versa."""
    st = np.arange(3 * 2 * 8, dtype=np.float32).reshape(2, 3, 8)
    p = tmp_path / "r.pgg"
    with open(p, "wb") as f:   # the reference's writer, restated
        f.write(b"PGG1")
        f.write(struct.pack("<II", 3, 2))
        f.write(st.astype("<f4").tobytes())
    np.testing.assert_array_equal(GB.checkpoint_load(p).stats, st)
