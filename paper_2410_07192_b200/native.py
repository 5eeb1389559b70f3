"""ctypes binding of libpipefill.so, the C ABI declared in include/pipefill.h.

This is the only way the package reaches the device: there is no CPU fallback.
If the shared library is missing or the device is not an sm_100 part, every
entry point raises :class:`NativeUnavailable` — loudly, at first use.
"""

from __future__ import annotations

import ctypes
import os
import re
from ctypes import POINTER, c_char_p, c_float, c_int, c_int64, c_uint32, c_uint64, c_void_p

LIB_NAME = "libpipefill.so"
# PF_LIB_PATH points at another build of the same ABI (diagnostic / A-B builds)
LIB_PATH = os.environ.get("PF_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)
HEADER_PATH = os.path.join(
    os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "pipefill.h"
)

PF_OK = 0
PF_ERR_INVALID = -1
PF_ERR_CUDA = -2
PF_ERR_UNSUPPORTED = -3
PF_ERR_OOM = -4

PF_EPI_BIAS = 1
PF_EPI_GELU = 2
PF_EPI_RESIDUAL = 4
PF_EPI_RELU = 8


class NativeUnavailable(RuntimeError):
    """libpipefill.so is missing or cannot run on this device."""


class PipeFillError(RuntimeError):
    """A C-ABI call returned a non-zero status."""

    def __init__(self, fn: str, code: int, message: str):
        super().__init__(f"{fn} failed with status {code}: {message}")
        self.fn = fn
        self.code = code


class ArenaExhausted(PipeFillError):
    """The fixed fill arena cannot satisfy an allocation (PF_ERR_OOM)."""


class PfCtl(ctypes.Structure):
    """Mirror of pf_ctl_t."""

    _fields_ = [("flag", c_void_p), ("abort", c_void_p), ("cursor", c_void_p)]


class SgdSegment(ctypes.Structure):
    """Mirror of pf_sgd_segment_t."""

    _fields_ = [("master", c_void_p), ("momentum", c_void_p), ("work", c_void_p), ("grad", c_void_p),
                ("n", ctypes.c_longlong), ("split_stride", ctypes.c_longlong), ("splits", c_int),
                ("grad_kind", c_int), ("weight_decay", c_float)]


_SIGNATURES: dict[str, tuple] = {
    "pf_abi_version": (c_int, []),
    "pf_last_error": (c_char_p, []),
    "pf_device_check": (c_int, [POINTER(c_int)]),
    "pf_arena_create": (c_int, [c_uint64, POINTER(c_void_p)]),
    "pf_arena_alloc": (c_int, [c_void_p, c_uint64, c_uint64, POINTER(c_void_p)]),
    "pf_arena_mark": (c_int, [c_void_p, POINTER(c_uint64)]),
    "pf_arena_release": (c_int, [c_void_p, c_uint64]),
    "pf_arena_reset": (c_int, [c_void_p]),
    "pf_arena_stats": (c_int, [c_void_p, POINTER(c_uint64), POINTER(c_uint64), POINTER(c_uint64)]),
    "pf_arena_base": (c_int, [c_void_p, POINTER(c_void_p)]),
    "pf_arena_destroy": (c_int, [c_void_p]),
    "pf_flag_create": (c_int, [POINTER(c_void_p)]),
    "pf_flag_destroy": (c_int, [c_void_p]),
    "pf_flag_write_on_stream": (c_int, [c_void_p, c_uint32, c_void_p]),
    "pf_flag_clear_at": (c_int, [c_void_p, c_void_p, c_uint64, c_void_p, c_void_p]),
    "pf_wait_until": (c_int, [c_void_p, c_uint64, c_void_p, c_void_p]),
    "pf_read_globaltimer": (c_int, [c_void_p, c_void_p]),
    "pf_sm_clock_probe": (c_int, [c_void_p, c_uint64, c_void_p]),
    "pf_flag_throttle_at": (c_int, [c_void_p, c_void_p, c_uint64, c_uint32, c_void_p]),
    "pf_host_alloc_pinned": (c_int, [c_uint64, POINTER(c_void_p)]),
    "pf_host_free_pinned": (c_int, [c_void_p]),
    "pf_stage_h2d": (c_int, [c_void_p, c_void_p, c_uint64, c_void_p]),
    "pf_stage_d2h": (c_int, [c_void_p, c_void_p, c_uint64, c_void_p]),
    "pf_gemm": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_uint32,
         POINTER(PfCtl), c_void_p],
    ),
    "pf_gemm_units": (c_int, [c_int, c_int, c_int, POINTER(c_uint32)]),
    "pf_layernorm": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_float,
         POINTER(PfCtl), c_void_p],
    ),
    "pf_rmsnorm": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_float, POINTER(PfCtl), c_void_p],
    ),
    "pf_norm_units": (c_int, [c_int, c_int, POINTER(c_uint32)]),
    "pf_softmax": (c_int, [c_void_p, c_void_p, c_int, c_int, c_float, POINTER(PfCtl), c_void_p]),
    "pf_softmax_units": (c_int, [c_int, c_int, POINTER(c_uint32)]),
    "pf_attention": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_float, POINTER(PfCtl),
         c_void_p],
    ),
    "pf_attention_units": (c_int, [c_int, c_int, c_int, c_int, POINTER(c_uint32)]),
    "pf_embedding_ln": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int,
         c_int, c_int, c_int, c_float, POINTER(PfCtl), c_void_p],
    ),
    "pf_copy": (c_int, [c_void_p, c_void_p, c_uint64, POINTER(PfCtl), c_void_p]),
    "pf_copy_units": (c_int, [c_uint64, POINTER(c_uint32)]),
    "pf_copy2d": (c_int, [c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64, POINTER(PfCtl),
                          c_void_p]),
    "pf_im2col": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int,
                          c_int, POINTER(PfCtl), c_void_p]),
    "pf_maxpool": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_int,
                           POINTER(PfCtl), c_void_p]),
    "pf_avgpool": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, POINTER(PfCtl), c_void_p]),
    "pf_image_units": (c_int, [c_int, ctypes.c_longlong, c_int, POINTER(c_uint32)]),
    "pf_chain_add_im2col": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int, c_int,
                                    c_int, c_int, c_int]),
    "pf_chain_add_maxpool": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int,
                                     c_int, c_int]),
    "pf_chain_add_avgpool": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int]),
    "pf_gemm_splitk": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int, POINTER(PfCtl),
                               c_void_p]),
    "pf_gemm_splitk_splits": (c_int, [c_int, c_int, POINTER(c_int)]),
    "pf_gemm_nn": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, POINTER(PfCtl), c_void_p]),
    "pf_gemm_splitk_tn": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int, POINTER(PfCtl),
                                  c_void_p]),
    "pf_chain_add_gemm_nn": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int]),
    "pf_chain_add_gemm_splitk_tn": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int]),
    "pf_colstats": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int,
                            POINTER(c_int), POINTER(PfCtl), c_void_p]),
    "pf_bn_finalize": (c_int, [c_void_p, c_int, c_int, c_int, c_void_p, c_void_p, c_float, c_void_p,
                               c_void_p, c_void_p, c_void_p, POINTER(PfCtl), c_void_p]),
    "pf_bn_bwd_finalize": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, POINTER(PfCtl), c_void_p]),
    "pf_bn_apply": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, ctypes.c_longlong, c_int, c_int,
                            POINTER(PfCtl), c_void_p]),
    "pf_bn_bwd_apply": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                c_void_p, c_void_p, c_void_p, c_int, c_int, POINTER(PfCtl), c_void_p]),
    "pf_transpose": (c_int, [c_void_p, c_void_p, c_int, c_int, POINTER(PfCtl), c_void_p]),
    "pf_col2im": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_int,
                          c_int, c_int, POINTER(PfCtl), c_void_p]),
    "pf_maxpool_bwd": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_int,
                               POINTER(PfCtl), c_void_p]),
    "pf_avgpool_bwd": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, POINTER(PfCtl), c_void_p]),
    "pf_maxpool_argmax": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_int,
                                  POINTER(PfCtl), c_void_p]),
    "pf_maxpool_bwd_argmax": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int, c_int,
                                      c_int, POINTER(PfCtl), c_void_p]),
    "pf_softmax_xent": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_float, POINTER(PfCtl),
                                c_void_p]),
    "pf_sgd_update": (c_int, [POINTER(SgdSegment), c_int, c_float, c_float, POINTER(PfCtl), c_void_p]),
    "pf_chain_add_gemm_splitk": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int]),
    "pf_chain_add_colstats": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                      c_int, c_int, POINTER(c_int)]),
    "pf_chain_add_bn_finalize": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_void_p, c_void_p, c_float,
                                         c_void_p, c_void_p, c_void_p, c_void_p]),
    "pf_chain_add_bn_bwd_finalize": (c_int, [c_void_p, c_void_p, c_int, c_int, c_void_p, c_void_p]),
    "pf_chain_add_bn_apply": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                      ctypes.c_longlong, c_int, c_int]),
    "pf_chain_add_bn_bwd_apply": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                          c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int]),
    "pf_chain_add_transpose": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int]),
    "pf_chain_add_col2im": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int,
                                    c_int, c_int, c_int, c_int]),
    "pf_chain_add_maxpool_bwd": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int,
                                         c_int, c_int, c_int]),
    "pf_chain_add_avgpool_bwd": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int]),
    "pf_chain_add_maxpool_argmax": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int,
                                            c_int, c_int, c_int]),
    "pf_chain_add_maxpool_bwd_argmax": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int,
                                                c_int, c_int, c_int, c_int]),
    "pf_chain_add_softmax_xent": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int,
                                          c_float]),
    "pf_chain_add_sgd": (c_int, [c_void_p, POINTER(SgdSegment), c_int, c_float, c_float]),
    "pf_gemm_f32": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_uint32,
                            POINTER(PfCtl), c_void_p]),
    "pf_layernorm_f32": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_float,
                                 POINTER(PfCtl), c_void_p]),
    "pf_embedding_ln_f32": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int,
                                    c_int, c_int, c_int, c_float, POINTER(PfCtl), c_void_p]),
    "pf_attention_f32": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_float, POINTER(PfCtl),
                                 c_void_p]),
    "pf_chain_add_gemm_f32": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int,
                                      c_int, c_uint32]),
    "pf_chain_add_layernorm_f32": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int,
                                           c_int, c_float]),
    "pf_chain_add_embedding_ln_f32": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                              c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_float]),
    "pf_chain_add_attention_f32": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_float]),
    "pf_chain_create": (c_int, [POINTER(c_void_p)]),
    "pf_chain_destroy": (c_int, [c_void_p]),
    "pf_chain_add_gemm": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int,
                                  c_int, c_int, c_uint32]),
    "pf_chain_add_layernorm": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                       c_int, c_int, c_float]),
    "pf_chain_add_rmsnorm": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int,
                                     c_float]),
    "pf_chain_add_softmax": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, c_float]),
    "pf_chain_add_attention": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int,
                                       c_int, c_float]),
    "pf_chain_add_embedding_ln": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                          c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int,
                                          c_float]),
    "pf_chain_add_copy": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64,
                                  c_int]),
    "pf_chain_size": (c_int, [c_void_p, POINTER(c_int)]),
    "pf_chain_set_timing": (c_int, [c_void_p, c_int]),
    "pf_chain_set_desc": (c_int, [c_void_p, c_void_p]),
    "pf_chain_set_stamps": (c_int, [c_void_p, c_void_p]),
    "pf_chain_build_graph": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, POINTER(c_int), c_int]),
    "pf_chain_graph_launch": (c_int, [c_void_p, c_void_p]),
    "pf_chain_node_elapsed": (c_int, [c_void_p, c_int, POINTER(c_float)]),
    "pf_chain_node_info": (c_int, [c_void_p, c_int, POINTER(c_uint32), POINTER(c_int)]),
    "pf_chain_launch": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int64,
                                c_int64, c_void_p]),
    "pf_chain_begin": (c_int, [c_void_p, c_int, c_void_p, c_void_p]),
    "pf_chain_end": (c_int, [c_void_p, c_void_p, c_void_p]),
    "pf_staging_create": (c_int, [POINTER(c_void_p), POINTER(c_void_p), POINTER(c_void_p), POINTER(c_uint64),
                                  c_int, c_void_p, c_void_p]),
    "pf_staging_launch": (c_int, [c_void_p, c_void_p]),
    "pf_staging_destroy": (c_int, [c_void_p]),
}

_lib: ctypes.CDLL | None = None


def declared_symbols(header: str = HEADER_PATH) -> list[str]:
    """Function names declared in include/pipefill.h (pf_* prototypes)."""
    text = open(header).read()
    return sorted(set(re.findall(r"\b(pf_[a-z0-9_]+)\s*\(", text)))


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load (once) and type the shared library; raise NativeUnavailable if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeUnavailable(
            f"{path} not found: build it with `make` (or __graft_entry__.build()); "
            "the fill executor has no CPU fallback"
        )
    try:
        lib = ctypes.CDLL(path)
    except OSError as exc:  # pragma: no cover - depends on the loader
        raise NativeUnavailable(f"cannot load {path}: {exc}") from exc
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    msg = load().pf_last_error()
    return msg.decode() if msg else ""


def check(fn: str, rc: int) -> None:
    if rc == PF_OK:
        return
    msg = last_error()
    if rc == PF_ERR_OOM:
        raise ArenaExhausted(fn, rc, msg)
    if rc == PF_ERR_UNSUPPORTED:
        raise NativeUnavailable(f"{fn}: {msg}")
    raise PipeFillError(fn, rc, msg)


def call(fn: str, *args) -> None:
    """Invoke a status-returning entry point and raise on failure."""
    check(fn, getattr(load(), fn)(*args))


_device_ok: set[int] = set()


def require_device() -> int:
    """Fail loudly unless the current CUDA device is an sm_100 part; returns SM count."""
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the fill executor runs only on B200 (sm_100a)")
    dev = torch.cuda.current_device()
    n = c_int(0)
    check("pf_device_check", load().pf_device_check(ctypes.byref(n)))
    _device_ok.add(dev)
    return n.value
