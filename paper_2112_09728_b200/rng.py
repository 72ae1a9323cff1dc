"""Per-lane PCG32 streams on the GPU; drop-in for pgtrace.rng
(pg/rng.py:25-55).  Same key chain, same outputs, bit for bit.

NumPy callers get NumPy back and their state arrays are advanced in place,
exactly like the reference; torch CUDA callers stay on the device.
"""

import numpy as np
import torch

from . import _conv, _lib

_MULT = np.uint64(6364136223846793005)
_INC = np.uint64(1442695040888963407)


def make_streams(seed, frame_index, lane_index, stream_id=0):
    """PCG32 state per lane (rng.py:25-39); same shape as lane_index."""
    torch_in = torch.is_tensor(lane_index)
    lanes = _conv.u64_to_dev(lane_index if torch_in else np.asarray(lane_index, dtype=np.uint64))
    shape = tuple(lanes.shape)
    lanes = lanes.reshape(-1)
    out = torch.empty_like(lanes)
    key = _lib.frame_key(seed, frame_index, stream_id)
    _lib.check(_lib.lib().pgg_make_streams(key, lanes.numel(), _lib.ptr(lanes), _lib.ptr(out), _lib.stream_ptr()))
    out = out.reshape(shape)
    if torch_in:
        return out
    return out.cpu().numpy().view(np.uint64).reshape(shape)


def _advance(state):
    """-> (device state view, device u32 outputs as int32, writeback)."""
    if torch.is_tensor(state):
        st = state.view(torch.int64) if state.dtype != torch.int64 else state
        if not (st.is_cuda and st.is_contiguous()):
            raise ValueError("state must be a contiguous CUDA tensor")
        out = torch.empty(st.shape, dtype=torch.int32, device=st.device)
        _lib.check(_lib.lib().pgg_next_u32(st.numel(), _lib.ptr(st), _lib.ptr(out), _lib.stream_ptr()))
        return out, None
    host = np.asarray(state)
    if host.dtype != np.uint64:
        raise TypeError("state must be a uint64 array")
    st = _conv.u64_to_dev(host).reshape(-1)
    out = torch.empty(st.shape, dtype=torch.int32, device=st.device)
    _lib.check(_lib.lib().pgg_next_u32(st.numel(), _lib.ptr(st), _lib.ptr(out), _lib.stream_ptr()))

    def writeback():
        host[...] = st.cpu().numpy().view(np.uint64).reshape(host.shape)
    return out.reshape(host.shape), writeback


def next_u32(state):
    """Advance every stream once, in place; uint32 outputs (rng.py:42-50)."""
    out, wb = _advance(state)
    if wb is None:
        return out
    wb()
    return out.cpu().numpy().view(np.uint32)


def next_f64(state):
    """Uniform float64 in [0, 1): next_u32 * 2^-32 (rng.py:53-55)."""
    out, wb = _advance(state)
    f = (out.to(torch.int64) & 0xFFFFFFFF).to(torch.float64) * (2.0 ** -32)
    if wb is None:
        return f
    wb()
    return f.cpu().numpy()
