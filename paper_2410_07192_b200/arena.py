"""The fill job's fixed device arena and its control words.

``Arena`` wraps pf_arena_t (one cudaMalloc outside torch's caching allocator,
bump allocation, PF_ERR_OOM instead of growth — SURVEY §2.1 "arena"). Device
tensors handed out are zero-copy torch views of arena memory (via
``__cuda_array_interface__``), so the kernels and torch agree on addresses
while the memory itself never enters torch's allocator: the main job's
allocator state is untouched by filling, and the fill job cannot grow past the
bytes the bubble characterization measured as free.
"""

from __future__ import annotations

import ctypes

import torch

from . import native

_TYPESTR = {
    torch.uint8: ("|u1", 1),
    torch.int16: ("<i2", 2),
    torch.int32: ("<i4", 4),
    torch.int64: ("<i8", 8),
    torch.float32: ("<f4", 4),
}


class _CAI:
    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {
            "shape": tuple(shape),
            "typestr": typestr,
            "data": (ptr, False),
            "version": 3,
            "strides": None,
        }


def device_view(ptr: int, shape, dtype: torch.dtype, device: torch.device | None = None) -> torch.Tensor:
    """Zero-copy torch tensor over raw device memory at `ptr`."""
    base_dtype = torch.int16 if dtype == torch.bfloat16 else dtype
    typestr, _ = _TYPESTR[base_dtype]
    t = torch.as_tensor(_CAI(ptr, shape, typestr), device=device or torch.device("cuda"))
    return t.view(torch.bfloat16) if dtype == torch.bfloat16 else t


def _nbytes(shape, dtype: torch.dtype) -> int:
    n = 1
    for s in shape:
        n *= int(s)
    return n * torch.empty((), dtype=dtype).element_size()


class Arena:
    """Fixed-size device pool for one fill executor (one per GPU)."""

    def __init__(self, capacity_bytes: int):
        native.require_device()
        self._h = ctypes.c_void_p()
        native.call("pf_arena_create", int(capacity_bytes), ctypes.byref(self._h))
        self.capacity = int(capacity_bytes)

    def alloc(self, shape, dtype: torch.dtype, align: int = 256) -> torch.Tensor:
        ptr = ctypes.c_void_p()
        native.call("pf_arena_alloc", self._h, _nbytes(shape, dtype), align, ctypes.byref(ptr))
        return device_view(ptr.value, shape, dtype)

    def mark(self) -> int:
        m = ctypes.c_uint64()
        native.call("pf_arena_mark", self._h, ctypes.byref(m))
        return m.value

    def release(self, mark: int) -> None:
        native.call("pf_arena_release", self._h, int(mark))

    def reset(self) -> None:
        native.call("pf_arena_reset", self._h)

    def stats(self) -> dict:
        cap, used, hw = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        native.call("pf_arena_stats", self._h, ctypes.byref(cap), ctypes.byref(used), ctypes.byref(hw))
        return {"capacity": cap.value, "used": used.value, "high_water": hw.value}

    def close(self) -> None:
        if self._h:
            native.call("pf_arena_destroy", self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass


class PinnedBuffer:
    """Page-locked host memory from pf_host_alloc_pinned, viewed as a CPU tensor."""

    def __init__(self, shape, dtype: torch.dtype):
        self.nbytes = _nbytes(shape, dtype)
        self._p = ctypes.c_void_p()
        native.call("pf_host_alloc_pinned", self.nbytes, ctypes.byref(self._p))
        raw = (ctypes.c_uint8 * self.nbytes).from_address(self._p.value)
        flat = torch.frombuffer(raw, dtype=torch.uint8)
        self.tensor = flat.view(dtype).view(*shape) if shape else flat.view(dtype)

    @property
    def ptr(self) -> int:
        return self._p.value

    def close(self) -> None:
        """Free the page-locked memory. `tensor` (and every view of it) is invalid after."""
        if self._p:
            native.call("pf_host_free_pinned", self._p)
            self._p = ctypes.c_void_p()
            self.tensor = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass
