"""Array plumbing at the API edge: NumPy in -> device -> NumPy out, or torch
CUDA in -> torch CUDA out.  No arithmetic happens here."""

import numpy as np
import torch

from . import _lib


def device():
    _lib.lib()  # raises PggUnavailable without CUDA / libpgg.so
    return torch.device("cuda", torch.cuda.current_device())


def is_torch(*xs):
    return any(torch.is_tensor(x) for x in xs)


def to_dev(a, dtype):
    """Contiguous CUDA tensor of `dtype` (torch dtype) from NumPy / torch / scalars."""
    if torch.is_tensor(a):
        return a.to(device=device(), dtype=dtype).contiguous()
    arr = np.ascontiguousarray(np.asarray(a))
    if arr.dtype == np.uint64:
        arr = arr.view(np.int64)
    return torch.from_numpy(arr).to(device=device(), dtype=dtype).contiguous()


def u64_to_dev(a):
    """uint64 PCG states -> int64 CUDA tensor with the same bits."""
    if torch.is_tensor(a):
        return a.to(device=device()).contiguous().view(torch.int64)
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.uint64))
    return torch.from_numpy(arr.view(np.int64)).to(device()).contiguous()


def back(t, like_torch, dtype=None):
    """Return a device tensor as the caller's array type."""
    if like_torch:
        return t
    out = t.detach().cpu().numpy()
    if dtype is not None:
        out = out.astype(dtype, copy=False)
    return out
