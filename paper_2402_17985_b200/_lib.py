"""Loader for the in-tree CUDA library ``libfqg.so`` (C ABI in include/fqg.h).

There is no CPU fallback: if the library is missing or fails to load, every
entry point raises. ``build()`` compiles it for sm_100a with nvcc.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FQG_LIB", os.path.join(PKG, "libfqg.so"))  # override: A/B builds
CSRC = os.path.join(PKG, "csrc")

# fqg_dtype
F64, F32, F16, BF16, I32, I8, I4, NONE = range(8)
# fqg_status
OK, ERR_INVALID, ERR_RUNTIME, ERR_CUDA, ERR_UNSUPPORTED = 0, -2, -3, -4, -5
SCALE_STATIC, SCALE_DYNAMIC = 0, 1

_lib = None


class FqgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class FqgInvalidArgument(FqgError, ValueError):
    """Maps std::invalid_argument of the reference."""


class FqgRuntimeError(FqgError):
    """Maps std::runtime_error of the reference."""


def build(jobs: int = 8) -> str:
    subprocess.run(["make", "-s", "-j", str(jobs), "-C", CSRC], check=True)
    return LIB_PATH


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FqgError(ERR_CUDA, f"{LIB_PATH} is not built (run __graft_entry__.build())")
        _lib = C.CDLL(LIB_PATH)
        _declare(_lib)
    return _lib


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = lib().fqg_last_error().decode(errors="replace")
    if rc == ERR_INVALID:
        raise FqgInvalidArgument(rc, msg)
    if rc == ERR_RUNTIME:
        raise FqgRuntimeError(rc, msg)
    raise FqgError(rc, msg)


P, I64, F64_, INT = C.c_void_p, C.c_int64, C.c_double, C.c_int


class LayerDesc(C.Structure):
    _fields_ = [
        ("bits", INT), ("k", I64), ("n", I64), ("smooth_scales", P), ("t_x", F64_),
        ("ext_x", P), ("block_x", I64), ("t_w", F64_), ("ext_w", P), ("block_w", I64),
        ("act_scale", F64_), ("weight_q", P), ("weight", P), ("w_scale", F64_),
        ("n_total", I64), ("n_begin", I64), ("a_format", INT), ("b_format", INT),
        ("scale_mode", INT), ("device", INT),
    ]


class LayerInfo(C.Structure):
    _fields_ = [
        ("bits", INT), ("a_format", INT), ("b_format", INT), ("scale_mode", INT),
        ("k", I64), ("n", I64), ("c1", I64), ("kp", I64), ("n_total", I64), ("n_begin", I64),
        ("t_x", F64_), ("t_w", F64_), ("act_scale", F64_), ("w_scale", F64_),
        ("weight_bytes", I64),
    ]


class SynthOpts(C.Structure):
    _fields_ = [
        ("rows", I64), ("samples", I64), ("in_channels", I64), ("out_channels", I64),
        ("outlier_fraction", F64_), ("outlier_min", F64_), ("outlier_max", F64_),
        ("channel_spread", F64_), ("act_tail_prob_max", F64_), ("act_tail_scale", F64_),
        ("weight_row_spread", F64_), ("seed", C.c_uint64),
    ]


# ncclAllGather-compatible collective (include/fqg.h fqg_allgather_fn)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p,
                           C.c_void_p)


class GemmPlan(C.Structure):
    _fields_ = [("kernel", INT), ("tile_m", INT), ("tile_n", INT), ("splits", INT), ("ctas", INT)]


class QuantOptions(C.Structure):
    _fields_ = [("mode", INT), ("alpha", F64_), ("beta", F64_), ("gamma", F64_), ("block", I64),
                ("bins", I64), ("smooth", INT), ("clip", INT), ("damping", F64_)]


# Every symbol include/fqg.h declares, with its ctypes signature.
SIGNATURES = {
    "fqg_last_error": (C.c_char_p, []),
    "fqg_version": (INT, []),
    "fqg_layer_create": (INT, [C.POINTER(LayerDesc), C.POINTER(P)]),
    "fqg_layer_destroy": (INT, [P]),
    "fqg_layer_get_info": (INT, [P, C.POINTER(LayerInfo)]),
    "fqg_layer_weight_q": (INT, [P, P, C.POINTER(F64_)]),
    "fqg_layer_forward": (INT, [P, P, INT, I64, P, INT, I64, P, INT, P, P]),
    "fqg_layer_run_host": (INT, [P, P, I64, P, C.POINTER(I64)]),
    "fqg_layer_quantize_acts": (INT, [P, P, INT, I64, P, P, P]),
    "fqg_layer_gemm": (INT, [P, P, I64, P, INT, I64, P, INT, P]),
    "fqg_layer_quantize_acts_ex": (INT, [P, P, INT, I64, P, P, P, P]),
    "fqg_layer_gemm_ex": (INT, [P, P, P, I64, P, INT, I64, P, INT, P]),
    "fqg_gemm": (INT, [P, INT, I64, P, INT, I64, I64, I64, I64, P, INT, I64, P, P, INT, P]),
    "fqg_gemm_plan": (INT, [I64, I64, I64, INT, INT, INT, C.POINTER(GemmPlan)]),
    "fqg_shard_bounds": (INT, [I64, INT, INT, C.POINTER(I64), C.POINTER(I64), C.POINTER(I64)]),
    "fqg_layer_forward_sharded": (INT, [P, P, INT, I64, P, INT, INT, INT, P, INT, P, P, P, P]),
    "fqg_quant_options_default": (None, [C.POINTER(QuantOptions)]),
    "fqg_calibrate": (INT, [P, I64, I64, P, I64, I64, C.POINTER(QuantOptions), INT, C.POINTER(P)]),
    "fqg_recipe_get": (INT, [P, C.POINTER(LayerDesc), C.POINTER(F64_), C.POINTER(F64_)]),
    "fqg_recipe_free": (INT, [P]),
    "fqg_model_load": (INT, [C.c_char_p, C.c_char_p, INT, INT, C.POINTER(P)]),
    "fqg_model_destroy": (INT, [P]),
    "fqg_model_num_layers": (INT, [P, C.POINTER(I64)]),
    "fqg_model_layer_name": (INT, [P, I64, C.c_char_p, I64]),
    "fqg_model_layer_recipe": (INT, [P, I64, C.POINTER(LayerDesc), C.POINTER(F64_),
                                     C.POINTER(F64_)]),
    "fqg_model_layer": (INT, [P, C.c_char_p, C.POINTER(P)]),
    "fqg_model_infer": (INT, [P, C.c_char_p, C.c_char_p, C.POINTER(I64), C.POINTER(I64)]),
    "fqg_hash64": (C.c_uint64, [P, C.c_size_t, C.c_uint64]),
    "fqg_build_flatten_plan": (INT, [P, I64, F64_, I64, P, P, C.POINTER(I64), C.POINTER(I64)]),
    "fqg_split_against_threshold": (None, [F64_, F64_, C.POINTER(I64), C.POINTER(F64_)]),
    "fqg_recipe_plan": (INT, [P, I64, I64, P, INT, F64_, F64_, I64, INT, INT, P,
                              C.POINTER(F64_), P, C.POINTER(I64), C.POINTER(F64_), P, I64,
                              C.POINTER(I64), C.POINTER(F64_)]),
    "fqg_collect_channel_maxes": (None, [P, I64, I64, P]),
    "fqg_gather_maps": (INT, [P, I64, I64, P, I64, P, P, P, C.POINTER(I64), I64]),
    "fqg_synth_default": (None, [C.POINTER(SynthOpts)]),
    "fqg_synthetic_layer": (INT, [C.POINTER(SynthOpts), I64, P, P, P, I64]),
}


def _declare(L: C.CDLL) -> None:
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name, None)
        if fn is None:
            continue  # reported by exported_symbols() / the ABI test
        fn.restype = res
        fn.argtypes = args


def exported_symbols() -> dict:
    """name -> bool (present in the loaded library)."""
    L = lib()
    return {name: hasattr(L, name) for name in SIGNATURES}
