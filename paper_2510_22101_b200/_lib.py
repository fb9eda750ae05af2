"""ctypes binding of libprefill_sm100.so (declared in include/prefill_sm100.h).

The library is built in-tree by ``__graft_entry__.build()`` / ``make -C
paper_2510_22101_b200/csrc``.  There is no fallback: if the shared object is
missing or cannot be loaded every product entry point raises
``NativeLibraryError``.
"""

from __future__ import annotations

import ctypes
import os

LIB_PATH = os.environ.get("PF_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                          "libprefill_sm100.so")   # override: A/B builds only

# Error codes (include/prefill_sm100.h)
PF_EARG, PF_ESHAPE, PF_ETMAP, PF_ECUDA, PF_EWORKSPACE, PF_ENONFINITE = -1, -2, -3, -4, -5, -6

EPI_BF16, EPI_ROPE_BF16, EPI_SWIGLU, EPI_RESID_ADD, EPI_RESID_ADD_NORM = 0, 1, 2, 3, 4

# Every symbol include/prefill_sm100.h declares (tests check the .so exports all of them).
EXPORTED_SYMBOLS = (
    "pf_model_create", "pf_model_destroy", "pf_workspace_bytes", "pf_score", "pf_score_host", "pf_score_capture",
    "pf_validate_packed", "pf_layer_tail", "pf_debug_set_mlp_stats",
    "pf_gemm_bf16", "pf_gemm_bf16_ex", "pf_embed", "pf_rmsnorm", "pf_prefix_attention", "pf_attention_last_rows", "pf_head_last_token",
    "pf_last_error", "pf_version", "pf_debug_set_trace", "pf_profile_enable", "pf_profile_read", "pf_profile_class_name",
    "pf_tokenize", "pf_tokenize_spans", "pf_tokenize_batch", "pf_pack_sizes", "pf_pack_requests",
)


class NativeLibraryError(RuntimeError):
    """libprefill_sm100.so is missing or failed to load (no CPU fallback exists)."""


class PfError(ValueError):
    """A C-ABI call returned a negative status (message from pf_last_error)."""

    def __init__(self, code: int, message: str):
        super().__init__(f"[{code}] {message}")
        self.code = code


class PfModelDesc(ctypes.Structure):
    _fields_ = [
        ("n_layers", ctypes.c_int), ("d_model", ctypes.c_int), ("n_heads", ctypes.c_int),
        ("n_kv_heads", ctypes.c_int), ("d_head", ctypes.c_int), ("d_ff", ctypes.c_int),
        ("d_ff_pad", ctypes.c_int), ("vocab_size", ctypes.c_int), ("max_seq", ctypes.c_int),
        ("rms_eps", ctypes.c_float),
        ("embedding", ctypes.c_void_p),
        ("w_qkv", ctypes.POINTER(ctypes.c_void_p)),
        ("w_o", ctypes.POINTER(ctypes.c_void_p)),
        ("w_gu", ctypes.POINTER(ctypes.c_void_p)),
        ("w_down", ctypes.POINTER(ctypes.c_void_p)),
        ("ln_final", ctypes.c_void_p),
        ("w_yes", ctypes.c_void_p),
        ("w_no", ctypes.c_void_p),
        ("rope_cos", ctypes.c_void_p),
        ("rope_sin", ctypes.c_void_p),
    ]


class PfGemmArgs(ctypes.Structure):
    _fields_ = [
        ("A", ctypes.c_void_p), ("lda", ctypes.c_int), ("B", ctypes.c_void_p), ("ldb", ctypes.c_int),
        ("C", ctypes.c_void_p), ("ldc", ctypes.c_int),
        ("M", ctypes.c_int), ("N", ctypes.c_int), ("K", ctypes.c_int), ("epilogue", ctypes.c_int),
        ("pos", ctypes.c_void_p), ("rope_cos", ctypes.c_void_p), ("rope_sin", ctypes.c_void_p),
        ("rope_heads", ctypes.c_int), ("rope_dh", ctypes.c_int),
        ("row_ss", ctypes.c_void_p), ("ss_ld", ctypes.c_longlong), ("ss_out", ctypes.c_void_p),
        ("xb", ctypes.c_void_p), ("ldxb", ctypes.c_int), ("inv_d", ctypes.c_float), ("eps", ctypes.c_float),
        ("rope_cs", ctypes.c_void_p),
    ]


class PfCapture(ctypes.Structure):
    """include/prefill_sm100.h pf_capture."""
    _fields_ = [("rows", ctypes.c_void_p), ("n_rows", ctypes.c_int), ("gains", ctypes.c_void_p),
                ("out", ctypes.c_void_p), ("out_layer_stride", ctypes.c_longlong)]


_lib = None

_P = ctypes.c_void_p
_I = ctypes.c_int
_F = ctypes.c_float
_SIGS = {
    "pf_model_create": (_I, [ctypes.POINTER(PfModelDesc), ctypes.POINTER(_P)]),
    "pf_model_destroy": (_I, [_P]),
    "pf_workspace_bytes": (ctypes.c_size_t, [_P, _I, _I]),
    "pf_score": (_I, [_P, _P, _P, _P, _I, _P, _I, _P, _I, _I, _P, ctypes.c_size_t, _P, _P, _P, _P]),
    "pf_score_capture": (_I, [_P, _P, _P, _P, _I, _P, _I, _P, _I, _I, _P, ctypes.c_size_t, _P, _P, _P,
                              ctypes.POINTER(PfCapture), _P]),
    "pf_debug_set_mlp_stats": (_I, [_P]),
    "pf_layer_tail": (_I, [_P, _I, _P, _P, _P, _P, _P, _P, _I, _P, ctypes.c_size_t, _P]),
    "pf_validate_packed": (_I, [_P, _P, _P, _P, _I, _P, _I, _P, _I, _I, _P, _P]),
    "pf_score_host": (_I, [_P, _P, _P, _P, _I, _P, _I, _P, _I, _I, _P, ctypes.c_size_t, _P, _P, _P]),
    "pf_gemm_bf16": (_I, [_P, _I, _P, _I, _P, _I, _I, _I, _I, _I, _P, _P, _P, _I, _P]),
    "pf_gemm_bf16_ex": (_I, [ctypes.POINTER(PfGemmArgs), _P]),
    "pf_embed": (_I, [_P, _P, _P, _P, _P, _P, _I, _I, _P]),
    "pf_rmsnorm": (_I, [_P, _P, _P, _I, _I, _F, _P]),
    "pf_prefix_attention": (_I, [_P, _P, _I, _I, _I, _I, _P, _P, _I, _P]),
    "pf_attention_last_rows": (_I, [_P, _P, _I, _I, _I, _P, _I, _P, _I, _I, _P, _P]),
    "pf_head_last_token": (_I, [_P, _P, _I, _I, _P, _P, _P, _F, _P, _P, _P, _P]),
    "pf_debug_set_trace": (_I, [_P, ctypes.c_uint]),
    "pf_tokenize": (_I, [ctypes.c_char_p, ctypes.c_size_t, _I, _I, _P, ctypes.c_int64, _P]),
    "pf_tokenize_spans": (_I, [ctypes.c_char_p, ctypes.c_size_t, _I, _I, _P, _P, ctypes.c_int64, _P]),
    "pf_tokenize_batch": (_I, [_P, _P, _I, _I, _I, _P, ctypes.c_int64, _P, _I]),
    "pf_pack_sizes": (_I, [_P, _P, _I, _P, _P, _P]),
    "pf_pack_requests": (_I, [_P, _P, _P, _I, _I, _P, _P, _P, _P, _P, _P, _P]),
    "pf_profile_enable": (_I, [_I]),
    "pf_profile_read": (_I, [_P, _P, _I]),
    "pf_profile_class_name": (ctypes.c_char_p, [_I]),
    "pf_last_error": (ctypes.c_char_p, []),
    "pf_version": (ctypes.c_char_p, []),
}


def load():
    """Load (once) and return the ctypes handle of libprefill_sm100.so."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryError(
            f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the scoring path)")
    try:
        lib = ctypes.CDLL(LIB_PATH)
    except OSError as e:  # pragma: no cover - depends on the box
        raise NativeLibraryError(f"failed to load {LIB_PATH}: {e}") from e
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc != 0:
        msg = load().pf_last_error().decode(errors="replace")
        raise PfError(rc, msg)


def version() -> str:
    return load().pf_version().decode()
