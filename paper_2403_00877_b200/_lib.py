"""ctypes binding of libdmt.so (the C ABI declared in include/dmt.h).

There is no CPU fallback: every op in this package goes through these entry
points and raises if the library or a CUDA device is missing.
"""

from __future__ import annotations

import ctypes as C
import os

import torch

from .errors import STATUS_ERRORS, TowersimError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DMT_LIB", os.path.join(_HERE, "libdmt.so"))  # DMT_LIB: A/B builds

DT_F32, DT_BF16, DT_F64, DT_F16 = 0, 1, 2, 3
POOL_NONE, POOL_SUM, POOL_MEAN = 0, 1, 2
EPI_NONE, EPI_BIAS, EPI_CROSS, EPI_ACC, EPI_DCN_BWD, EPI_DCN_FINAL = 0, 1, 2, 3, 4, 5
EPI_BIAS_RELU, EPI_RELU_BWD = 6, 7
GEMM_TRANS_A, GEMM_TRANS_B, GEMM_AUX2_ACCUM, GEMM_SCALE_ACC = 1, 2, 4, 8
GEMM_NO_PREFETCH, GEMM_BN_SHIFT, GEMM_CLUSTER, GEMM_SINGLE_CTA = 16, 8, 32, 64  # tuning overrides
GEMM_NO_TMA_STORE = 0x1000
GEMM_MAX_PAIRS = 4
GEMM_MAX_OUT_GROUPS = 8
GEMM_MAX_COL_GROUPS = 32
MAX_PEER_SRCS = 8  # DMT_MAX_PEER_SRCS (include/dmt.h)
OPT_SGD, OPT_ROWWISE_ADAGRAD = 0, 1
EBIT_INDEX, EBIT_BAGLEN = 1, 2

TORCH_DT = {torch.float32: DT_F32, torch.bfloat16: DT_BF16, torch.float64: DT_F64, torch.float16: DT_F16}
POOL_CODE = {"none": POOL_NONE, "sum": POOL_SUM, "mean": POOL_MEAN}

vp, i32, i64, f32, sz = C.c_void_p, C.c_int32, C.c_int64, C.c_float, C.c_size_t


class LookupSegment(C.Structure):
    _fields_ = [
        ("weights", vp), ("out", vp), ("state", vp),
        ("ld", i64), ("out_ld", i64), ("bag_begin", i64), ("row_begin", i64), ("key_base", i64),
        ("rows", i32), ("width", i32), ("nbags", i32), ("pooling", i32), ("row_filter", i32), ("table_rows", i32),
    ]


class SlotDst(C.Structure):
    _fields_ = [("len", vp), ("val", vp), ("room", i64)]


class AssembleBlock(C.Structure):
    _fields_ = [("dst_col", i64), ("width", i32), ("nsrc", i32), ("first_src", i32), ("groups", C.c_uint32)]


class Src(C.Structure):
    _fields_ = [("ptr", vp), ("ld", i64)]


class Copy(C.Structure):
    _fields_ = [("src", vp), ("dst", vp), ("bytes", i64)]


class Copy2D(C.Structure):
    _fields_ = [("src", vp), ("dst", vp), ("src_ld", i64), ("dst_ld", i64), ("rows", i64), ("width", i64)]


class GemmArgs(C.Structure):
    _fields_ = [
        ("a", vp), ("b", vp), ("d", vp), ("bias", vp), ("x0", vp), ("xl", vp), ("aux", vp), ("c", vp),
        ("aux2", vp),
        ("m", i64), ("n", i64), ("k", i64),
        ("lda", i64), ("ldb", i64), ("ld_d", i64), ("ld_x", i64),
        ("rows_per_group", i64), ("ld_group", i64),
        ("beta", f32), ("alpha", f32), ("in_dtype", i32), ("out_dtype", i32), ("epilogue", i32), ("flags", i32),
        ("npairs", i32), ("pad_", i32), ("pair_g", vp * GEMM_MAX_PAIRS), ("pair_u", vp * GEMM_MAX_PAIRS),
        ("colsum_part", vp), ("ksplit", i32), ("n_out_groups", i32), ("splitk_ws", vp),
        ("out_group", vp * GEMM_MAX_OUT_GROUPS),
        ("n_col_groups", i32), ("col_group_width", i32), ("col_group", vp * GEMM_MAX_COL_GROUPS),
        ("col_group_ld", i64 * GEMM_MAX_COL_GROUPS),
    ]


_SIGS = {
    "dmt_version": (C.c_char_p, []),
    "dmt_last_error": (C.c_char_p, []),
    "dmt_enable_peer_access": (C.c_int, [C.c_int]),
    "dmt_ipc_export": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_int64)]),
    "dmt_ipc_open": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "dmt_ipc_close": (C.c_int, [C.c_void_p]),
    "dmt_lengths_to_offsets_workspace_size": (sz, [i64]),
    "dmt_lengths_to_offsets": (C.c_int, [vp, i64, vp, vp, vp]),
    "dmt_kjt_bucketize": (C.c_int, [vp, vp, vp, i32, i32, vp, vp, vp, vp, vp]),
    "dmt_kjt_slot_offsets": (C.c_int, [vp, i32, i32, vp, vp, vp]),
    "dmt_kjt_compact": (C.c_int, [vp, vp, i32, i32, vp, vp, vp]),
    "dmt_kjt_bucketize_peer": (C.c_int, [vp, vp, vp, i32, i32, vp, vp, vp]),
    "dmt_kjt_check_capacity": (C.c_int, [vp, i32, i32, vp, vp, vp]),
    "dmt_pooled_lookup_fwd": (C.c_int, [vp, vp, i32, vp, vp, i32, vp, vp]),
    "dmt_pooled_lookup_bwd_workspace_size": (sz, [i64, i64, i64]),
    "dmt_pooled_lookup_bwd": (C.c_int, [vp, vp, i32, vp, vp, i64, i64, i32, i32, f32, f32, vp, sz, vp]),
    "dmt_pooled_lookup_bwd_prepare": (C.c_int, [vp, vp, i32, vp, vp, i64, i64, i32, vp, sz, vp]),
    "dmt_pooled_lookup_bwd_apply": (C.c_int, [vp, vp, i32, i64, i64, i32, i32, f32, f32, vp, sz, vp]),
    "dmt_assemble": (C.c_int, [vp, i32, i32, vp, i64, vp, i64, i32, vp]),
    "dmt_batched_copy": (C.c_int, [vp, i32, i64, vp]),
    "dmt_batched_copy2d": (C.c_int, [vp, i32, i32, i64, vp]),
    "dmt_gemm": (C.c_int, [vp, vp]),
    "dmt_gemm_ex": (C.c_int, [vp, vp, vp, vp]),
    "dmt_split_tf32": (C.c_int, [vp, vp, vp, i64, vp]),
    "dmt_transpose": (C.c_int, [vp, i64, i64, i64, vp, i64, i32, vp]),
    "dmt_column_sum_workspace_size": (sz, [i64, i64]),
    "dmt_column_sum": (C.c_int, [vp, i64, i64, i64, vp, i32, vp, sz, vp]),
    "dmt_gemm_colsum_rows": (i64, [i64]),
    "dmt_bce_with_logits": (C.c_int, [vp, vp, i64, i32, f32, vp, vp, vp]),
    "dmt_column_sum_parts": (C.c_int, [vp, i64, i64, vp, vp]),
    "dmt_cross_bwd_pointwise": (C.c_int, [vp, vp, vp, vp, vp, i64, i32, vp]),
    "dmt_dcn_dx0_term": (C.c_int, [vp, vp, vp, i64, i32, i32, vp]),
    "dmt_dcn_side_fused_workspace_size": (sz, [i64, i64, i32]),
    "dmt_dcn_side_fused": (C.c_int, [C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), i32, i64,
                                     i64, vp, C.POINTER(C.c_void_p), i32, vp, sz, vp]),
    "dmt_sgd_dense": (C.c_int, [vp, vp, i64, f32, i32, vp]),
    "dmt_peer_sum_sgd": (C.c_int, [vp, C.POINTER(C.c_void_p), i32, i64, f32, i32, vp]),
    "dmt_peer_barrier": (C.c_int, [vp, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), i32, vp, vp]),
    "dmt_convert": (C.c_int, [vp, i32, vp, i32, i64, vp]),
    "dmt_relu_bwd": (C.c_int, [vp, vp, vp, i64, i32, vp]),
    "dmt_dot_interaction_fwd": (C.c_int, [vp, i64, vp, i64, i32, i32, i64, vp, i64, i32, vp]),
    "dmt_dot_interaction_bwd": (C.c_int, [vp, i64, vp, i64, vp, i64, i32, i32, i64, vp, i64, vp, i64, i32, vp]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load_library(require_cuda: bool = True):
    """Load libdmt.so once.  Raises (never falls back) if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise TowersimError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2403_00877_b200.build` "
                "(there is no CPU fallback)"
            )
        lib = C.CDLL(LIB_PATH)
        ab_build = "DMT_LIB" in os.environ  # an older A/B build may lack newer entry points
        for name, (res, args) in _SIGS.items():
            if ab_build and not hasattr(lib, name):
                continue
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    if require_cuda and not torch.cuda.is_available():
        raise TowersimError("libdmt needs a CUDA (sm_100a) device; none is visible (no CPU fallback)")
    return _lib


def lib():
    return load_library(True)


CALLS = [0]  # libdmt entry-point calls (each launches >= 1 kernel); read by bench.py


def check(status: int, what: str) -> None:
    CALLS[0] += 1
    if status != 0:
        cls = STATUS_ERRORS.get(status, TowersimError)
        extra = ""
        if status == -10:
            extra = ": " + _lib.dmt_last_error().decode()
        raise cls(f"{what} failed with libdmt status {status}{extra}")


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def struct_array(ctype, items):
    arr = (ctype * max(1, len(items)))()
    for i, it in enumerate(items):
        arr[i] = it
    return arr


def upload_structs(arr, n: int, device) -> torch.Tensor:
    """Copy a ctypes struct array to a device byte tensor (pinned staging)."""
    nbytes = C.sizeof(arr) if n else 0
    host = torch.empty(max(nbytes, 1), dtype=torch.uint8, pin_memory=True)
    if nbytes:
        C.memmove(host.data_ptr(), C.addressof(arr), nbytes)
    dev = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)
    dev.copy_(host, non_blocking=True)
    return dev
