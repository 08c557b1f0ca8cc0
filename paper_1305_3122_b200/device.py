"""Device plumbing: CUDA availability, result blocks, and host<->device staging.

PyTorch is used only as the allocator and stream provider; every computation goes through
libfemasm_b200.so.  ``require_cuda()`` is called by every compute entry point so a missing
GPU or library fails loudly instead of falling back to the CPU.
"""

from __future__ import annotations

import numpy as np

from . import _lib


def require_cuda():
    """Return the torch module after checking that CUDA and the library are usable."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_1305_3122_b200 needs a CUDA device (B200, sm_100a); none is visible")
    _lib.load_library()
    return torch


def device():
    torch = require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


class ResultBlock:
    """A device ``fa_result`` block plus its host mirror."""

    def __init__(self):
        torch = require_cuda()
        self.dev = torch.zeros(_lib.RESULT_WORDS, dtype=torch.int64, device=device())

    @property
    def ptr(self) -> int:
        return self.dev.data_ptr()

    def fetch(self) -> _lib.FaResult:
        return _lib.result_from_words(self.dev.cpu().numpy())


def to_device(arr: np.ndarray, dtype=None):
    """Upload a numpy array (contiguous) to the current CUDA device."""
    torch = require_cuda()
    a = np.ascontiguousarray(arr if dtype is None else arr.astype(dtype, copy=False))
    if not a.flags.writeable:  # frozen Mesh arrays: torch.from_numpy needs a writable buffer
        a = a.copy()
    return torch.from_numpy(a).to(device(), non_blocking=False)


def connectivity_int32(connectivity: np.ndarray) -> np.ndarray:
    conn = np.asarray(connectivity)
    if conn.size and (conn.max() >= 2**31 - 1 or conn.min() < -(2**31)):
        raise ValueError("connectivity ids do not fit the 32-bit device layout")
    return np.ascontiguousarray(conn, dtype=np.int32)
