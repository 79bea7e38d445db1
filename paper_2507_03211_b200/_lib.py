"""ctypes binding of libzo_b200.so (the C ABI in include/zo_b200.h).

The library is the product path: there is no Python or CPU fallback.  If
it is missing or the device is not sm_100, ``lib()`` raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import CudaError, raise_for

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ZO_B200_LIB", os.path.join(_HERE, "lib", "libzo_b200.so"))

# status codes / enums (include/zo_b200.h)
ZO_OK = 0
ZO_Z_PHILOX, ZO_Z_ORACLE = 0, 1
ZO_SHADOW_BF16, ZO_SHADOW_F32, ZO_SHADOW_NONE = 0, 1, 2
ZO_PU_UPDATE, ZO_PU_SHADOW_A, ZO_PU_SHADOW_B, ZO_PU_FILL = 1, 2, 4, 8
ZO_EPI_F32, ZO_EPI_BIAS_BF16, ZO_EPI_BIAS_GELU_BF16, ZO_EPI_BIAS_RESID_F32, ZO_EPI_CE = 0, 1, 2, 3, 4
ZO_EPI_BIAS_RELU_BF16 = 5
ZO_GEMM_B_KMAJOR = 0x100


class ZoSegment(C.Structure):
    _fields_ = [("src", C.c_int64), ("rows", C.c_int64), ("cols", C.c_int64), ("dst", C.c_int64),
                ("dst_ld", C.c_int64), ("kind", C.c_int32), ("reserved", C.c_int32)]


class ZoStepScalars(C.Structure):
    _fields_ = [("seed_cur", C.c_uint64), ("seed_prev", C.c_uint64), ("lr_g_prev", C.c_double),
                ("pending", C.c_int64)]


P = C.c_void_p
I64 = C.c_int64
I32 = C.c_int32
D = C.c_double
U32 = C.c_uint32
U64 = C.c_uint64

# name -> (restype, argtypes); every symbol include/zo_b200.h declares
SIGNATURES = {
    "zo_version": (C.c_char_p, []),
    "zo_last_error": (C.c_char_p, []),
    "zo_device_check": (C.c_int, [C.c_int]),
    "zo_perturb_update": (C.c_int, [P, I64, P, P, I32, I64, P, P, P, P, D, D, U32, P, I32, P, P, I64, P]),
    "zo_perturb_tile_elems": (I64, []),
    "zo_embed_fwd": (C.c_int, [P, I64, P, I64, P, I64, I64, I64, I64, D, P, I32, P, I64, P, I64, P, P]),
    "zo_layernorm_fwd": (C.c_int, [P, I64, P, P, I64, I64, P, I64, P]),
    "zo_layernorm_fwd_split": (C.c_int, [P, I64, P, P, P, P, I64, I64, I64, P, I64, P]),
    "zo_gemm_bf16_split": (C.c_int, [P, I64, P, P, I64, I64, I64, I64, I64, I32, P, P, P, I64, P, P, P, P, P]),
    "zo_gemm_bf16": (C.c_int, [P, I64, P, I64, I64, I64, I64, I32, P, P, I64, P, P, P, P, P]),
    "zo_gemm_ce_tiles": (I64, [I64]),
    "zo_attn_causal_fwd": (C.c_int, [P, I64, I64, I64, I64, I64, P, I64, P]),
    "zo_gemm_f32": (C.c_int, [P, I64, P, I64, I64, I64, I64, I32, P, P, I64, P]),
    "zo_attn_causal_fwd_f32": (C.c_int, [P, I64, I64, I64, I64, I64, P, I64, P]),
    "zo_layernorm_fwd_f32": (C.c_int, [P, I64, P, P, I64, I64, P, I64, P]),
    "zo_ce_rows_f32": (C.c_int, [P, I64, I64, I64, P, P, P, I64, P, P]),
    "zo_ce_finalize": (C.c_int, [P, P, I64, I64, P, P, P, P]),
    "zo_grad_finalize": (C.c_int, [P, P, D, D, P, P, P]),
    "zo_grad_finalize_groups": (C.c_int, [P, I32, I32, I32, I32, I32, I32, D, D, P, P, P]),
    "zo_hash_u64": (C.c_int, [P, I64, P, P, P]),
    "zo_graph_begin": (C.c_int, [P]),
    "zo_copy_async": (C.c_int, [P, P, I64, P]),
    "zo_graph_end": (C.c_int, [P, P]),
    "zo_graph_launch": (C.c_int, [P, P]),
    "zo_graph_destroy": (C.c_int, [P]),
    "zo_planes_join": (C.c_int, [P, P, P, I64, P]),
    "zo_planes_split": (C.c_int, [P, P, P, I64, P]),
    "zo_philox_normals": (C.c_int, [U64, I64, I64, P, P]),
}

_lock = threading.Lock()
_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load the shared library and bind every exported symbol (no device
    needed; used by the CPU ABI test)."""
    if not os.path.exists(path):
        raise CudaError(f"native library not built: {path} (run paper_2507_03211_b200.build_lib)")
    dll = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(dll, name)
        fn.restype = res
        fn.argtypes = args
    return dll


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                dll = load()
                import torch

                if not torch.cuda.is_available():
                    raise CudaError("paper_2507_03211_b200 needs a CUDA device (B200, sm_100a); none visible")
                dev = torch.cuda.current_device()
                rc = dll.zo_device_check(dev)
                if rc:
                    raise_for(rc, dll.zo_last_error().decode())
                _lib = dll
    return _lib


def check(rc: int) -> None:
    if rc:
        raise_for(rc, _lib.zo_last_error().decode() if _lib is not None else f"status {rc}")


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
