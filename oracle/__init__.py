"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the FlattenQuant hot path.

Two checkers, both plain CPU code:

* ``Port``: ``oracle/fq_oracle.c``, a literal C restatement of the reference
  hot path (``/root/reference/proj/core/src/{flatten,quantize,smoothing,
  calibration,pipeline}.cpp``), built to ``oracle/_build/libfq_oracle.so``.
* ``Ref``: the UNMODIFIED reference ``fq_core`` compiled from its own sources by
  ``oracle/Makefile`` into ``oracle/_ref/libfq_ref.so`` (C ABI in
  ``oracle/ref_shim.cpp``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
may import this package; the product (``paper_2402_17985_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libfq_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfq_ref.so")
REF_SRC = "/root/reference/proj/core"

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
P = C.c_void_p
I64 = C.c_int64
F64 = C.c_double


class OracleError(RuntimeError):
    pass


class InvalidArgument(OracleError, ValueError):
    """std::invalid_argument in the reference."""


class ReferenceRuntimeError(OracleError):
    """std::runtime_error in the reference."""


def _check(rc: int, what: str, msg: str = "") -> None:
    if rc == 0:
        return
    text = f"{what}: {msg}" if msg else what
    if rc == -2:
        raise InvalidArgument(text)
    if rc == -3:
        raise ReferenceRuntimeError(text)
    raise OracleError(f"{text} (rc={rc})")


def build(ref: bool = True) -> None:
    """Compile the checkers (``make -C oracle``); the reference only if present."""
    import subprocess

    targets = ["port"]
    if ref and os.path.isdir(REF_SRC):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


@dataclass
class Layer:
    """A frozen recipe (reference ``LayerQuantConfig``, pipeline.hpp:37-49)."""

    bits: int
    s: np.ndarray  # [K] f64 smoothing scales
    t_x: float
    e_x: np.ndarray  # [K] int64 plan_x extensions
    t_w: float
    e_w: np.ndarray  # [C1] int64 plan_w extensions
    wq: np.ndarray  # [K', N] int32 weight_q (row-major, as the reference)
    s_w: float
    act_scale: float
    block: int = 32
    extra: dict = field(default_factory=dict)

    @property
    def k(self) -> int:
        return int(self.e_x.shape[0])

    @property
    def n(self) -> int:
        return int(self.wq.shape[1])

    @property
    def c1(self) -> int:
        return padded_width(self.e_x, self.block)

    @property
    def kp(self) -> int:
        return padded_width(self.e_w, self.block)


def padded_width(e: np.ndarray, block: int = 32) -> int:
    w = int(e.shape[0] + int(np.sum(e)))
    return (w + block - 1) // block * block


class Port:
    """ctypes view of ``oracle/_build/libfq_oracle.so`` (the C restatement)."""

    class _L(C.Structure):
        _fields_ = [
            ("bits", C.c_int), ("k", I64), ("n", I64), ("s", P), ("t_x", F64), ("t_w", F64),
            ("e_x", P), ("e_w", P), ("c1", I64), ("kp", I64), ("block", I64), ("wq", P),
            ("s_w", F64), ("act_scale", F64),
        ]

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build(ref=False)
        self.lib = C.CDLL(path)
        L = self.lib
        L.fqo_split_against_threshold.argtypes = [F64, F64, C.POINTER(I64), C.POINTER(F64)]
        L.fqo_build_flatten_plan.argtypes = [_f64p, I64, F64, I64, _i64p, P, C.POINTER(I64),
                                             C.POINTER(I64)]
        L.fqo_flatten_columns.argtypes = [_f64p, I64, I64, F64, _i64p, I64, C.c_int, _f64p,
                                          C.POINTER(I64)]
        L.fqo_flatten_rows.argtypes = [_f64p, I64, I64, F64, _i64p, I64, C.c_int, _f64p]
        L.fqo_repeat_channels.argtypes = [_f64p, I64, I64, _i64p, I64, _f64p]
        L.fqo_repeat_columns.argtypes = [_f64p, I64, I64, _i64p, I64, _f64p]
        L.fqo_quantize_per_tensor.argtypes = [_f64p, I64, C.c_int, F64, _i32p, C.POINTER(F64)]
        L.fqo_int_matmul_raw.argtypes = [_i32p, I64, I64, C.c_int, _i32p, I64, C.c_int, _i64p]
        L.fqo_accumulator_bound_ok.argtypes = [I64, I64, I64]
        L.fqo_derive_truncation.argtypes = [_f64p, I64, F64, C.c_int, C.POINTER(F64)]
        L.fqo_smoothing_scales.argtypes = [_f64p, _f64p, I64, F64, _f64p]
        L.fqo_collect_channel_maxes.argtypes = [_f64p, I64, I64, I64, _f64p]
        L.fqo_quantize_layer_pinned.argtypes = [_f64p, I64, I64, _f64p, I64, I64, C.c_int, F64,
                                                F64, I64, C.c_int, C.c_int,
                                                C.POINTER(Port._L)]
        L.fqo_layer_free.argtypes = [C.POINTER(Port._L)]
        L.fqo_run_layer.argtypes = [C.POINTER(Port._L), _f64p, I64, _f64p, C.POINTER(I64), P, P]
        L.fqo_quantize_acts.argtypes = [C.POINTER(Port._L), _f64p, I64, P, C.POINTER(I64)]

    # -- flatten.cpp -----------------------------------------------------
    def split(self, a: float, t: float) -> tuple[int, float]:
        c, r = I64(), F64()
        self.lib.fqo_split_against_threshold(a, t, C.byref(c), C.byref(r))
        return c.value, r.value

    def build_plan(self, maxes, t: float, block: int = 32):
        maxes = np.ascontiguousarray(maxes, np.float64)
        e = np.zeros(max(1, maxes.shape[0]), np.int64)
        off = np.zeros_like(e)
        c, p = I64(), I64()
        _check(self.lib.fqo_build_flatten_plan(maxes, maxes.shape[0], t, block, e,
                                                off.ctypes.data, C.byref(c), C.byref(p)),
               "build_flatten_plan")
        return e, off, c.value, p.value

    def flatten_columns(self, x, t, e, block=32, strict=False):
        x = np.ascontiguousarray(x, np.float64)
        e = np.ascontiguousarray(e, np.int64)
        out = np.zeros((x.shape[0], padded_width(e, block)))
        sat = I64()
        _check(self.lib.fqo_flatten_columns(x, x.shape[0], x.shape[1], t, e, block, int(strict),
                                            out, C.byref(sat)), "flatten_tensor")
        return out, sat.value

    def flatten_rows(self, w, t, e, block=32):
        w = np.ascontiguousarray(w, np.float64)
        e = np.ascontiguousarray(e, np.int64)
        out = np.zeros((padded_width(e, block), w.shape[1]))
        _check(self.lib.fqo_flatten_rows(w, w.shape[0], w.shape[1], t, e, block, 1, out),
               "flatten_rows")
        return out

    def repeat_channels(self, w, e, block=32):
        w = np.ascontiguousarray(w, np.float64)
        e = np.ascontiguousarray(e, np.int64)
        out = np.zeros((padded_width(e, block), w.shape[1]))
        self.lib.fqo_repeat_channels(w, w.shape[0], w.shape[1], e, block, out)
        return out

    def repeat_columns(self, x, e, block=32):
        x = np.ascontiguousarray(x, np.float64)
        e = np.ascontiguousarray(e, np.int64)
        out = np.zeros((x.shape[0], padded_width(e, block)))
        self.lib.fqo_repeat_columns(x, x.shape[0], x.shape[1], e, block, out)
        return out

    # -- quantize.cpp ----------------------------------------------------
    def quantize(self, m, bits, scale=None):
        m = np.ascontiguousarray(m, np.float64)
        q = np.zeros(m.shape, np.int32)
        s = F64()
        _check(self.lib.fqo_quantize_per_tensor(m.reshape(-1), m.size, bits,
                                                0.0 if scale is None else scale,
                                                q.reshape(-1), C.byref(s)), "quantize_per_tensor")
        return q, s.value

    def int_matmul_raw(self, qx, qw, bits_x=8, bits_w=8):
        qx = np.ascontiguousarray(qx, np.int32)
        qw = np.ascontiguousarray(qw, np.int32)
        acc = np.zeros((qx.shape[0], qw.shape[1]), np.int64)
        _check(self.lib.fqo_int_matmul_raw(qx, qx.shape[0], qx.shape[1], bits_x, qw, qw.shape[1],
                                           bits_w, acc), "int_matmul_raw")
        return acc

    # -- calibration / smoothing ----------------------------------------
    def derive_truncation(self, maxes, beta=1.3, clip=True):
        maxes = np.ascontiguousarray(maxes, np.float64)
        t = F64()
        _check(self.lib.fqo_derive_truncation(maxes, maxes.shape[0], beta, int(clip),
                                              C.byref(t)), "derive_truncation")
        return t.value

    def smoothing_scales(self, act_max, w_max, alpha=0.5):
        a = np.ascontiguousarray(act_max, np.float64)
        w = np.ascontiguousarray(w_max, np.float64)
        s = np.zeros_like(a)
        _check(self.lib.fqo_smoothing_scales(a, w, a.shape[0], alpha, s), "smoothing_scales")
        return s

    # -- pipeline.cpp ----------------------------------------------------
    def quantize_layer(self, w, calib, bits, alpha=0.5, beta=1.3, block=32, smooth=True,
                       clip=True) -> Layer:
        w = np.ascontiguousarray(w, np.float64)
        calib = np.ascontiguousarray(calib, np.float64)
        if calib.ndim == 2:
            calib = calib[None]
        L = Port._L()
        _check(self.lib.fqo_quantize_layer_pinned(w, w.shape[0], w.shape[1], calib.reshape(-1),
                                                  calib.shape[0], calib.shape[1], bits, alpha,
                                                  beta, block, int(smooth), int(clip),
                                                  C.byref(L)), "quantize_layer")
        k, n, c1, kp = L.k, L.n, L.c1, L.kp
        arr = lambda p, t, cnt: np.ctypeslib.as_array(C.cast(p, C.POINTER(t)), (cnt,)).copy()
        out = Layer(bits=L.bits, s=arr(L.s, F64, k), t_x=L.t_x, e_x=arr(L.e_x, I64, k),
                    t_w=L.t_w, e_w=arr(L.e_w, I64, c1),
                    wq=arr(L.wq, C.c_int32, kp * n).reshape(kp, n), s_w=L.s_w,
                    act_scale=L.act_scale, block=int(L.block))
        self.lib.fqo_layer_free(C.byref(L))
        return out

    def _as_struct(self, layer: Layer, keep: list):
        s = np.ascontiguousarray(layer.s, np.float64)
        ex = np.ascontiguousarray(layer.e_x, np.int64)
        ew = np.ascontiguousarray(layer.e_w, np.int64)
        wq = np.ascontiguousarray(layer.wq, np.int32)
        keep += [s, ex, ew, wq]
        return Port._L(layer.bits, layer.k, layer.n, _ptr(s), layer.t_x, layer.t_w, _ptr(ex),
                       _ptr(ew), layer.c1, layer.kp, layer.block, _ptr(wq), layer.s_w,
                       layer.act_scale)

    def quantize_acts(self, layer: Layer, x):
        """The activation half of run_layer (pipeline.cpp:164-167): (qx int32 [M,K'], sat)."""
        x = np.ascontiguousarray(x, np.float64)
        if x.shape[1] != layer.k:
            raise InvalidArgument("run_layer: input channel count does not match recipe")
        keep: list = []
        L = self._as_struct(layer, keep)
        qx = np.zeros((x.shape[0], layer.kp), np.int32)
        sat = I64()
        _check(self.lib.fqo_quantize_acts(C.byref(L), x, x.shape[0], _ptr(qx), C.byref(sat)),
               "quantize_acts")
        return qx, sat.value

    @staticmethod
    def exact_acc(qx, wq):
        """int_matmul_raw (quantize.cpp:166-188) for full-size checks: an f64 BLAS
        product of the integer operands. Exact, in any summation order, because
        every partial sum is an integer below 2^53 (|acc| <= K' * 127^2)."""
        assert qx.shape[1] * 127 * 127 < 2 ** 53
        return (qx.astype(np.float64) @ wq.astype(np.float64)).astype(np.int64)

    def run_layer(self, layer: Layer, x, debug: bool = False):
        """Returns (y f64 [M,N], saturation) or, with debug, (y, sat, qx int32, acc int64)."""
        x = np.ascontiguousarray(x, np.float64)
        if x.shape[1] != layer.k:
            raise InvalidArgument("run_layer: input channel count does not match recipe")
        keep: list = []
        L = self._as_struct(layer, keep)
        m = x.shape[0]
        y = np.zeros((m, layer.n))
        sat = I64()
        qx = np.zeros((m, layer.kp), np.int32) if debug else None
        acc = np.zeros((m, layer.n), np.int64) if debug else None
        _check(self.lib.fqo_run_layer(C.byref(L), x, m, y, C.byref(sat),
                                      None if qx is None else _ptr(qx),
                                      None if acc is None else _ptr(acc)), "run_layer")
        if debug:
            return y, sat.value, qx, acc
        return y, sat.value


class Ref:
    """ctypes view of ``oracle/_ref/libfq_ref.so``: the unmodified reference."""

    class SynthOpts(C.Structure):
        _fields_ = [("rows", I64), ("samples", I64), ("in_channels", I64),
                    ("out_channels", I64), ("outlier_fraction", F64), ("outlier_min", F64),
                    ("outlier_max", F64), ("channel_spread", F64), ("act_tail_prob_max", F64),
                    ("act_tail_scale", F64), ("weight_row_spread", F64), ("seed", C.c_uint64)]

    class QOpts(C.Structure):
        _fields_ = [("mode", C.c_int), ("alpha", F64), ("beta", F64), ("gamma", F64),
                    ("block", I64), ("bins", I64), ("damping", F64), ("smooth", C.c_int),
                    ("clip", C.c_int)]

    class Info(C.Structure):
        _fields_ = [("bits", C.c_int), ("K", I64), ("N", I64), ("C1", I64), ("Kp", I64),
                    ("cext_x", I64), ("cext_w", I64), ("T_x", F64), ("T_w", F64),
                    ("act_scale", F64), ("s_w", F64), ("kl_ratio_act", F64),
                    ("kl_ratio_w", F64)]

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO) or os.path.isdir(REF_SRC)

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            build(ref=True)
        self.lib = C.CDLL(path)
        L = self.lib
        L.fqref_last_error.restype = C.c_char_p
        L.fqref_synthetic_layer.argtypes = [C.POINTER(Ref.SynthOpts), I64, P, P, P, P, P]
        L.fqref_quantize_layer.argtypes = [_f64p, I64, I64, _f64p, I64, I64,
                                           C.POINTER(Ref.QOpts), C.POINTER(P)]
        L.fqref_layer_from_arrays.argtypes = [C.c_int, I64, I64, _f64p, F64, _i64p, I64, F64,
                                              _i64p, I64, _i32p, F64, F64, C.POINTER(P)]
        L.fqref_layer_free.argtypes = [P]
        L.fqref_write_model.argtypes = [P, P, I64, C.c_char_p, C.c_char_p]
        L.fqref_write_f64_archive.argtypes = [C.c_char_p, P, P, P, P, I64]
        L.fqref_infer.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p,
                                  C.POINTER(I64), C.POINTER(I64)]
        L.fqref_layer_info_get.argtypes = [P, C.POINTER(Ref.Info)]
        L.fqref_layer_arrays.argtypes = [P, P, P, P, P]
        L.fqref_run_layer.argtypes = [P, _f64p, I64, _f64p, C.POINTER(I64), C.c_int]
        L.fqref_quantized_acts.argtypes = [P, _f64p, I64, _i32p, C.POINTER(I64)]
        L.fqref_int_matmul_raw.argtypes = [_i32p, I64, I64, C.c_int, _i32p, I64, C.c_int, _i64p]
        L.fqref_build_flatten_plan.argtypes = [_f64p, I64, F64, I64, _i64p, P, C.POINTER(I64),
                                               C.POINTER(I64)]
        L.fqref_split_against_threshold.argtypes = [F64, F64, C.POINTER(I64), C.POINTER(F64)]
        L.fqref_flatten_tensor.argtypes = [_f64p, I64, I64, F64, _i64p, I64, C.c_int, _f64p,
                                           C.POINTER(I64)]
        L.fqref_flatten_rows.argtypes = [_f64p, I64, I64, F64, _i64p, I64, _f64p]
        L.fqref_repeat.argtypes = [_f64p, I64, I64, F64, _i64p, I64, C.c_int, _f64p]
        L.fqref_quantize_per_tensor.argtypes = [_f64p, I64, I64, C.c_int, P, _i32p,
                                                C.POINTER(F64)]
        L.fqref_collect_channel_maxes.argtypes = [_f64p, I64, I64, I64, _f64p]
        L.fqref_derive_truncation.argtypes = [_f64p, I64, F64, C.c_int, C.POINTER(F64)]
        L.fqref_smoothing_scales.argtypes = [_f64p, _f64p, I64, F64, _f64p]
        L.fqref_default_synth_opts.argtypes = [C.POINTER(Ref.SynthOpts)]
        L.fqref_default_qopts.argtypes = [C.POINTER(Ref.QOpts)]

    def _c(self, rc, what):
        _check(rc, what, self.lib.fqref_last_error().decode() if rc else "")

    # -- synthetic.cpp ---------------------------------------------------
    def synth_opts(self, **kw) -> "Ref.SynthOpts":
        o = Ref.SynthOpts()
        self.lib.fqref_default_synth_opts(C.byref(o))
        for k, v in kw.items():
            setattr(o, k, v)
        return o

    def synthetic_layer(self, index: int = 0, **kw):
        """fq::make_synthetic_layer -> (weight [K,N], calib [S,R,K], test_input [R,K], outliers)."""
        o = self.synth_opts(**kw)
        k, n, r, s = o.in_channels, o.out_channels, o.rows, o.samples
        w = np.zeros((k, n))
        calib = np.zeros((s, r, k))
        x = np.zeros((r, k))
        idx = np.zeros(k, np.int64)
        cnt = I64()
        self._c(self.lib.fqref_synthetic_layer(C.byref(o), index, _ptr(w), _ptr(calib), _ptr(x),
                                               _ptr(idx), C.byref(cnt)), "synthetic_layer")
        return w, calib, x, idx[: cnt.value].copy()

    # -- pipeline.cpp ----------------------------------------------------
    def write_model(self, layers, names, recipe_path: str, qmodel_path: str) -> None:
        """cmd_quantize's outputs (flattenquant_cli.cpp:199-238): recipe JSON via the
        reference's schemas.cpp, "<layer>.qweight" FQTA archive via archive.cpp."""
        hs = (P * len(layers))(*[l.h for l in layers])
        ns = (C.c_char_p * len(names))(*[n.encode() for n in names])
        self._c(self.lib.fqref_write_model(hs, ns, len(layers), recipe_path.encode(),
                                           qmodel_path.encode()), "write_model")

    def write_f64_archive(self, path: str, tensors: dict) -> None:
        items = [(k, np.ascontiguousarray(v, np.float64)) for k, v in tensors.items()]
        n = len(items)
        names = (C.c_char_p * n)(*[k.encode() for k, _ in items])
        data = (P * n)(*[v.ctypes.data for _, v in items])
        rows = (I64 * n)(*[v.shape[0] for _, v in items])
        cols = (I64 * n)(*[v.shape[1] for _, v in items])
        self._c(self.lib.fqref_write_f64_archive(path.encode(), names, data, rows, cols, n),
                "write_f64_archive")

    def infer(self, qmodel_path: str, recipe_path: str, input_path: str, out_path: str):
        """The reference cmd_infer: -> (saturated elements, tensors run)."""
        sat, ran = I64(), I64()
        self._c(self.lib.fqref_infer(qmodel_path.encode(), recipe_path.encode(),
                                     input_path.encode(), out_path.encode(), C.byref(sat),
                                     C.byref(ran)), "infer")
        return sat.value, ran.value

    def quantize_layer(self, w, calib, mode: int = 1, **kw) -> "RefLayer":
        w = np.ascontiguousarray(w, np.float64)
        calib = np.ascontiguousarray(calib, np.float64)
        if calib.ndim == 2:
            calib = calib[None]
        o = Ref.QOpts()
        self.lib.fqref_default_qopts(C.byref(o))
        o.mode = mode
        for k, v in kw.items():
            setattr(o, k, v)
        h = P()
        self._c(self.lib.fqref_quantize_layer(w, w.shape[0], w.shape[1], calib.reshape(-1),
                                              calib.shape[0], calib.shape[1], C.byref(o),
                                              C.byref(h)), "quantize_layer")
        return RefLayer(self, h)

    def layer_from(self, layer: Layer) -> "RefLayer":
        h = P()
        self._c(self.lib.fqref_layer_from_arrays(
            layer.bits, layer.k, layer.n, np.ascontiguousarray(layer.s, np.float64), layer.t_x,
            np.ascontiguousarray(layer.e_x, np.int64), layer.block, layer.t_w,
            np.ascontiguousarray(layer.e_w, np.int64), layer.block,
            np.ascontiguousarray(layer.wq, np.int32), layer.s_w, layer.act_scale, C.byref(h)),
            "layer_from_arrays")
        return RefLayer(self, h)

    def int_matmul_raw(self, qx, qw, bits_x=8, bits_w=8):
        qx = np.ascontiguousarray(qx, np.int32)
        qw = np.ascontiguousarray(qw, np.int32)
        acc = np.zeros((qx.shape[0], qw.shape[1]), np.int64)
        self._c(self.lib.fqref_int_matmul_raw(qx, qx.shape[0], qx.shape[1], bits_x, qw,
                                              qw.shape[1], bits_w, acc), "int_matmul_raw")
        return acc

    # -- flatten.cpp / quantize.cpp -------------------------------------
    def build_plan(self, maxes, t, block=32):
        maxes = np.ascontiguousarray(maxes, np.float64)
        e = np.zeros(max(1, maxes.shape[0]), np.int64)
        off = np.zeros_like(e)
        c, p = I64(), I64()
        self._c(self.lib.fqref_build_flatten_plan(maxes, maxes.shape[0], t, block, e,
                                                  off.ctypes.data, C.byref(c), C.byref(p)),
                "build_flatten_plan")
        return e, off, c.value, p.value

    def split(self, a, t):
        c, r = I64(), F64()
        self.lib.fqref_split_against_threshold(a, t, C.byref(c), C.byref(r))
        return c.value, r.value

    def flatten_columns(self, x, t, e, block=32, strict=False):
        x = np.ascontiguousarray(x, np.float64)
        e = np.ascontiguousarray(e, np.int64)
        out = np.zeros((x.shape[0], padded_width(e, block)))
        sat = I64()
        self._c(self.lib.fqref_flatten_tensor(x, x.shape[0], x.shape[1], t, e, block,
                                              0 if strict else 1, out, C.byref(sat)),
                "flatten_tensor")
        return out, sat.value

    def flatten_rows(self, w, t, e, block=32):
        w = np.ascontiguousarray(w, np.float64)
        e = np.ascontiguousarray(e, np.int64)
        out = np.zeros((padded_width(e, block), w.shape[1]))
        self._c(self.lib.fqref_flatten_rows(w, w.shape[0], w.shape[1], t, e, block, out),
                "flatten_rows")
        return out

    def repeat_channels(self, w, e, block=32):
        w = np.ascontiguousarray(w, np.float64)
        e = np.ascontiguousarray(e, np.int64)
        out = np.zeros((padded_width(e, block), w.shape[1]))
        self._c(self.lib.fqref_repeat(w, w.shape[0], w.shape[1], 1.0, e, block, 0, out),
                "repeat_channels")
        return out

    def repeat_columns(self, x, e, block=32):
        x = np.ascontiguousarray(x, np.float64)
        e = np.ascontiguousarray(e, np.int64)
        out = np.zeros((x.shape[0], padded_width(e, block)))
        self._c(self.lib.fqref_repeat(x, x.shape[0], x.shape[1], 1.0, e, block, 1, out),
                "repeat_columns")
        return out

    def quantize(self, m, bits, scale=None):
        m = np.ascontiguousarray(m, np.float64)
        m2 = m.reshape(1, -1) if m.ndim == 1 else m
        q = np.zeros(m2.shape, np.int32)
        s = F64()
        sc = F64(scale) if scale is not None else None
        self._c(self.lib.fqref_quantize_per_tensor(m2, m2.shape[0], m2.shape[1], bits,
                                                   None if sc is None else C.addressof(sc), q,
                                                   C.byref(s)), "quantize_per_tensor")
        return q.reshape(m.shape), s.value

    def collect_channel_maxes(self, calib):
        calib = np.ascontiguousarray(calib, np.float64)
        out = np.zeros(calib.shape[-1])
        self._c(self.lib.fqref_collect_channel_maxes(calib.reshape(-1), calib.shape[0],
                                                     calib.shape[1], calib.shape[2], out),
                "collect_channel_maxes")
        return out

    def derive_truncation(self, maxes, beta=1.3, clip=True):
        maxes = np.ascontiguousarray(maxes, np.float64)
        t = F64()
        self._c(self.lib.fqref_derive_truncation(maxes, maxes.shape[0], beta, int(clip),
                                                 C.byref(t)), "derive_truncation")
        return t.value

    def smoothing_scales(self, act_max, w_max, alpha=0.5):
        a = np.ascontiguousarray(act_max, np.float64)
        w = np.ascontiguousarray(w_max, np.float64)
        s = np.zeros_like(a)
        self._c(self.lib.fqref_smoothing_scales(a, w, a.shape[0], alpha, s), "smoothing_scales")
        return s


class RefLayer:
    """Owns a reference ``LayerQuantConfig``."""

    def __init__(self, ref: Ref, handle: P):
        self.ref, self.h = ref, handle
        info = Ref.Info()
        ref._c(ref.lib.fqref_layer_info_get(handle, C.byref(info)), "layer_info")
        self.info = info

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.fqref_layer_free(self.h)
            self.h = None

    def to_layer(self) -> Layer:
        i = self.info
        s = np.zeros(i.K)
        ex = np.zeros(i.K, np.int64)
        ew = np.zeros(i.C1, np.int64)
        wq = np.zeros((i.Kp, i.N), np.int32)
        self.ref._c(self.ref.lib.fqref_layer_arrays(self.h, _ptr(s), _ptr(ex), _ptr(ew),
                                                    _ptr(wq)), "layer_arrays")
        return Layer(bits=i.bits, s=s, t_x=i.T_x, e_x=ex, t_w=i.T_w, e_w=ew, wq=wq, s_w=i.s_w,
                     act_scale=i.act_scale,
                     extra={"kl_ratio_act": i.kl_ratio_act, "kl_ratio_w": i.kl_ratio_w})

    def run_layer(self, x, nthreads: int = 1):
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros((x.shape[0], self.info.N))
        sat = I64()
        self.ref._c(self.ref.lib.fqref_run_layer(self.h, x, x.shape[0], y, C.byref(sat),
                                                 nthreads), "run_layer")
        return y, sat.value

    def quantized_acts(self, x):
        x = np.ascontiguousarray(x, np.float64)
        q = np.zeros((x.shape[0], self.info.Kp), np.int32)
        sat = I64()
        self.ref._c(self.ref.lib.fqref_quantized_acts(self.h, x, x.shape[0], q, C.byref(sat)),
                    "quantized_acts")
        return q, sat.value
