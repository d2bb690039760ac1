"""B200-native FlattenQuant linear-layer hot path (arXiv 2402.17985).

Python mirror of the reference operator API (``/root/reference/proj/core``,
namespace ``fq``) over the C ABI of ``libfqg.so`` (include/fqg.h). Names,
argument meaning and error behaviour follow the reference:

=====================================  =========================================
reference (file:line)                  here
=====================================  =========================================
``fq::FlattenPlan`` flatten.hpp:17-33  :class:`FlattenPlan`
``fq::build_flatten_plan`` :36-37       :func:`build_flatten_plan`
``fq::split_against_threshold`` :46     :func:`split_against_threshold`
``fq::LayerQuantConfig`` pipeline.hpp   :class:`LayerQuantConfig`
``fq::quantize_layer`` pipeline.hpp:77  :func:`quantize_layer` (bits pinned)
``fq::run_layer`` pipeline.hpp:83-84    :func:`run_layer` / :meth:`Layer.run_layer`
``fq::make_synthetic_layer``            :func:`synthetic_layer`
=====================================  =========================================

``std::invalid_argument`` surfaces as :class:`FqgInvalidArgument` (a
``ValueError``), ``std::runtime_error`` as :class:`FqgRuntimeError`. Every
compute call runs the sm_100a kernels; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from ._lib import (BF16, F16, F32, F64, I4, I8, I32, NONE, SCALE_DYNAMIC, SCALE_STATIC,  # noqa
                   FqgError, FqgInvalidArgument, FqgRuntimeError, check, lib)

__all__ = [
    "FlattenPlan", "build_flatten_plan", "split_against_threshold", "LayerQuantConfig",
    "Layer", "Model", "calibrate", "quantize_layer", "run_layer", "synthetic_layer", "FqgError",
    "FqgInvalidArgument", "FqgRuntimeError",
]

_f64 = lambda a: np.ascontiguousarray(a, dtype=np.float64)  # noqa: E731
_i64 = lambda a: np.ascontiguousarray(a, dtype=np.int64)  # noqa: E731


@dataclass
class FlattenPlan:
    """fq::FlattenPlan (flatten.hpp:17-33)."""

    threshold: float
    extensions: np.ndarray
    ext_offset: np.ndarray
    c_extend: int
    padded_width: int
    block: int = 32

    def channels(self) -> int:
        return int(self.extensions.shape[0])

    def width(self) -> int:
        return self.channels() + self.c_extend

    def identity(self) -> bool:
        return self.c_extend == 0

    def flatten_ratio(self) -> float:
        return self.c_extend / self.channels()

    def slot_of(self, j: int) -> list:
        first = self.channels() + int(self.ext_offset[j])
        return [j] + [first + q for q in range(int(self.extensions[j]))]

    @staticmethod
    def from_extensions(threshold: float, extensions, block: int = 32) -> "FlattenPlan":
        e = _i64(extensions)
        off = np.concatenate([[0], np.cumsum(e)[:-1]]).astype(np.int64)
        c = int(e.sum())
        w = e.shape[0] + c
        return FlattenPlan(float(threshold), e, off, c, (w + block - 1) // block * block, block)


def split_against_threshold(abs_value: float, threshold: float) -> tuple[int, float]:
    """fq::split_against_threshold (flatten.cpp:8-15): (count, remainder)."""
    c, r = C.c_int64(), C.c_double()
    lib().fqg_split_against_threshold(abs_value, threshold, C.byref(c), C.byref(r))
    return c.value, r.value


def build_flatten_plan(channel_maxes, threshold: float, block: int = 32) -> FlattenPlan:
    """fq::build_flatten_plan (flatten.cpp:17-45)."""
    m = _f64(channel_maxes)
    k = m.shape[0]
    e = np.zeros(max(k, 1), np.int64)
    off = np.zeros_like(e)
    c, p = C.c_int64(), C.c_int64()
    check(lib().fqg_build_flatten_plan(m.ctypes.data, k, threshold, block, e.ctypes.data,
                                       off.ctypes.data, C.byref(c), C.byref(p)))
    return FlattenPlan(float(threshold), e[:k], off[:k], c.value, p.value, block)


@dataclass
class LayerQuantConfig:
    """The frozen recipe fields fq::run_layer reads (pipeline.hpp:37-49).

    ``weight_q`` is the reference layout: int32 [K', N] row-major, with scale
    ``w_scale``. Alternatively ``weight`` (f64 [K, N]) lets the device run the
    offline weight tail of quantize_layer (pipeline.cpp:100,114-120,139-150).
    """

    bits: int
    smooth_scales: np.ndarray
    plan_x: FlattenPlan
    plan_w: FlattenPlan
    act_scale: float
    weight_q: Optional[np.ndarray] = None
    w_scale: float = 0.0
    weight: Optional[np.ndarray] = None
    extra: dict = field(default_factory=dict)

    @property
    def k(self) -> int:
        return self.plan_x.channels()

    @property
    def n(self) -> int:
        src = self.weight_q if self.weight_q is not None else self.weight
        return int(src.shape[1])


_DT = {}


def _torch_dtype_code(t) -> int:
    import torch

    global _DT
    if not _DT:
        _DT = {torch.float64: F64, torch.float32: F32, torch.float16: F16,
               torch.bfloat16: BF16, torch.int32: I32}
    return _DT[t.dtype]


class Layer:
    """A device-resident quantized layer (one ``fqg_layer_t``)."""

    def __init__(self, cfg: LayerQuantConfig, device: int = 0, a_format: int = I8,
                 b_format: int = I8, scale_mode: int = SCALE_STATIC,
                 n_begin: int = 0, n: Optional[int] = None):
        self.cfg = cfg
        n_total = cfg.n
        n = n_total - n_begin if n is None else n
        keep = [_f64(cfg.smooth_scales), _i64(cfg.plan_x.extensions), _i64(cfg.plan_w.extensions)]
        d = _lib.LayerDesc()
        d.bits, d.k, d.n = cfg.bits, cfg.k, n
        d.smooth_scales = keep[0].ctypes.data
        d.t_x, d.ext_x, d.block_x = cfg.plan_x.threshold, keep[1].ctypes.data, cfg.plan_x.block
        d.t_w, d.ext_w, d.block_w = cfg.plan_w.threshold, keep[2].ctypes.data, cfg.plan_w.block
        d.act_scale = cfg.act_scale
        if cfg.weight_q is not None:
            wq = np.ascontiguousarray(cfg.weight_q, np.int32)
            keep.append(wq)
            d.weight_q, d.w_scale = wq.ctypes.data, cfg.w_scale
        else:
            w = _f64(cfg.weight)
            keep.append(w)
            d.weight = w.ctypes.data
        d.n_total, d.n_begin = n_total, n_begin
        d.a_format, d.b_format, d.scale_mode, d.device = a_format, b_format, scale_mode, device
        h = C.c_void_p()
        check(lib().fqg_layer_create(C.byref(d), C.byref(h)))
        self._h = h
        self.device = device
        info = _lib.LayerInfo()
        check(lib().fqg_layer_get_info(h, C.byref(info)))
        self.info = info

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().fqg_layer_destroy(h)
            except Exception:
                pass
            self._h = None

    # -- properties -----------------------------------------------------
    @property
    def k(self) -> int:
        return self.info.k

    @property
    def n(self) -> int:
        return self.info.n

    @property
    def kp(self) -> int:
        return self.info.kp

    @property
    def w_scale(self) -> float:
        return self.info.w_scale

    def weight_q(self) -> np.ndarray:
        """int32 [K', n] row-major (reference weight_q layout) read back from HBM."""
        out = np.zeros((self.kp, self.n), np.int32)
        s = C.c_double()
        check(lib().fqg_layer_weight_q(self._h, out.ctypes.data, C.byref(s)))
        return out

    # -- compute ----------------------------------------------------------
    def run_layer(self, x) -> tuple[np.ndarray, int]:
        """fq::run_layer(cfg, x, saturation) on host f64 buffers (pipeline.hpp:84)."""
        x = _f64(x)
        if x.ndim != 2 or x.shape[1] != self.k:
            raise FqgInvalidArgument(-2, "run_layer: input channel count does not match recipe")
        y = np.zeros((x.shape[0], self.n))
        sat = C.c_int64()
        check(lib().fqg_layer_run_host(self._h, x.ctypes.data, x.shape[0], y.ctypes.data,
                                       C.byref(sat)))
        return y, sat.value

    def forward(self, x, out_dtype=None, bias=None, saturation=None, out=None, stream=None):
        """Device-resident forward on torch CUDA tensors: y [M, n]."""
        import torch

        if x.dim() != 2 or x.shape[1] != self.k:
            raise FqgInvalidArgument(-2, "run_layer: input channel count does not match recipe")
        x = x.contiguous()
        m = x.shape[0]
        if out is None:
            out = torch.empty((m, self.n), dtype=out_dtype or torch.float16, device=x.device)
        st = stream if stream is not None else torch.cuda.current_stream(x.device).cuda_stream
        check(lib().fqg_layer_forward(
            self._h, x.data_ptr(), _torch_dtype_code(x), m, out.data_ptr(),
            _torch_dtype_code(out), out.stride(0),
            bias.data_ptr() if bias is not None else None,
            _torch_dtype_code(bias) if bias is not None else NONE,
            saturation.data_ptr() if saturation is not None else None, st))
        return out

    def quantize_acts(self, x, saturation=None):
        """K1 alone: quantized operand [M, K'] int8 (or [M, K'/2] packed int4)."""
        import torch

        x = x.contiguous()
        cols = self.kp // 2 if self.info.a_format == I4 else self.kp
        q = torch.empty((x.shape[0], cols), dtype=torch.int8, device=x.device)
        check(lib().fqg_layer_quantize_acts(
            self._h, x.data_ptr(), _torch_dtype_code(x), x.shape[0], q.data_ptr(),
            saturation.data_ptr() if saturation is not None else None,
            torch.cuda.current_stream(x.device).cuda_stream))
        return q

    def quantize_acts_rowsum(self, x, saturation=None):
        """K1 with the operand row sums the biased-int4 GEMM epilogue uses."""
        import torch

        x = x.contiguous()
        cols = self.kp // 2 if self.info.a_format == I4 else self.kp
        q = torch.empty((x.shape[0], cols), dtype=torch.int8, device=x.device)
        rowsum = torch.empty(x.shape[0], dtype=torch.int32, device=x.device)
        check(lib().fqg_layer_quantize_acts_ex(
            self._h, x.data_ptr(), _torch_dtype_code(x), x.shape[0], q.data_ptr(),
            rowsum.data_ptr(), saturation.data_ptr() if saturation is not None else None,
            torch.cuda.current_stream(x.device).cuda_stream))
        return q, rowsum

    def gemm_rows(self, q, rowsum, r0: int, rows: int, out, bias=None):
        """K4 on operand rows [r0, r0 + rows) into `out` ([rows, n] view, any row stride)."""
        import torch

        check(lib().fqg_layer_gemm_ex(
            self._h, q[r0:].data_ptr(), rowsum[r0:].data_ptr(), rows, out.data_ptr(),
            _torch_dtype_code(out), out.stride(0), bias.data_ptr() if bias is not None else None,
            _torch_dtype_code(bias) if bias is not None else NONE,
            torch.cuda.current_stream(q.device).cuda_stream))
        return out

    def gemm(self, q, out_dtype=None, bias=None, out=None):
        """K4 alone on an operand from :meth:`quantize_acts`."""
        import torch

        m = q.shape[0]
        if out is None:
            out = torch.empty((m, self.n), dtype=out_dtype or torch.float16, device=q.device)
        check(lib().fqg_layer_gemm(
            self._h, q.data_ptr(), m, out.data_ptr(), _torch_dtype_code(out), out.stride(0),
            bias.data_ptr() if bias is not None else None,
            _torch_dtype_code(bias) if bias is not None else NONE,
            torch.cuda.current_stream(q.device).cuda_stream))
        return out


def calibrate(weight, calib, mode: int = 2, device: int = 0, **opts):
    """fq::quantize_layer (pipeline.cpp:76-152, modes O1 = 1 / O2 = 2) with the
    calibration scans and the KL bit selection on the device. weight f64 [K, N],
    calib f64 [samples, rows, K]. Returns (LayerQuantConfig with weight = W, info)
    where info holds the KL ratios and the recipe's s_w."""
    o = _lib.QuantOptions()
    lib().fqg_quant_options_default(C.byref(o))
    o.mode = mode
    for key, v in opts.items():
        setattr(o, key, v)
    w = _f64(weight)
    c = _f64(calib)
    if c.ndim == 2:
        c = c[None]
    h = C.c_void_p()
    check(lib().fqg_calibrate(w.ctypes.data, w.shape[0], w.shape[1], c.ctypes.data, c.shape[0],
                              c.shape[1], C.byref(o), device, C.byref(h)))
    try:
        d = _lib.LayerDesc()
        ka, kw = C.c_double(), C.c_double()
        check(lib().fqg_recipe_get(h, C.byref(d), C.byref(ka), C.byref(kw)))
        k = d.k
        arr = lambda p, t, n: np.ctypeslib.as_array((t * n).from_address(p)).copy()  # noqa: E731
        e_x = arr(d.ext_x, C.c_int64, k)
        px = FlattenPlan.from_extensions(d.t_x, e_x, d.block_x)
        e_w = arr(d.ext_w, C.c_int64, px.padded_width)
        pw = FlattenPlan.from_extensions(d.t_w, e_w, d.block_w)
        if d.weight_q:  # O3: the device GPTQ weight_q
            wq = arr(d.weight_q, C.c_int32, pw.padded_width * d.n).reshape(pw.padded_width, d.n)
            cfg = LayerQuantConfig(bits=d.bits, smooth_scales=arr(d.smooth_scales, C.c_double, k),
                                   plan_x=px, plan_w=pw, act_scale=d.act_scale, weight_q=wq,
                                   w_scale=d.w_scale)
        else:
            cfg = LayerQuantConfig(bits=d.bits, smooth_scales=arr(d.smooth_scales, C.c_double, k),
                                   plan_x=px, plan_w=pw, act_scale=d.act_scale, weight=w)
        info = {"kl_ratio_act": ka.value, "kl_ratio_w": kw.value, "w_scale": d.w_scale}
        cfg.extra.update(info)
        return cfg, info
    finally:
        lib().fqg_recipe_free(h)


class Model:
    """Recipe JSON + FQTA quantized archive -> device layers (the CLI's
    load_recipes, flattenquant_cli.cpp:241-252); ``infer`` is cmd_infer
    (flattenquant_cli.cpp:254-281) on archives. device < 0: parse only."""

    def __init__(self, recipe_path: str, qmodel_path: Optional[str], device: int = 0,
                 a_format: int = I8):
        h = C.c_void_p()
        check(lib().fqg_model_load(recipe_path.encode(),
                                   qmodel_path.encode() if qmodel_path else None, device,
                                   a_format, C.byref(h)))
        self._h = h
        n = C.c_int64()
        check(lib().fqg_model_num_layers(h, C.byref(n)))
        self.names = []
        for i in range(n.value):
            buf = C.create_string_buffer(1024)
            check(lib().fqg_model_layer_name(h, i, buf, 1024))
            self.names.append(buf.value.decode())

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().fqg_model_destroy(h)
            except Exception:
                pass
            self._h = None

    def recipe(self, i: int) -> dict:
        """The parsed recipe of layer i (plain numpy copies)."""
        d = _lib.LayerDesc()
        ka, kw = C.c_double(), C.c_double()
        check(lib().fqg_model_layer_recipe(self._h, i, C.byref(d), C.byref(ka), C.byref(kw)))
        k = d.k
        c1 = -(-(k + int(np.ctypeslib.as_array((C.c_int64 * k).from_address(d.ext_x)).sum()))
               // d.block_x) * d.block_x
        arr = lambda p, t, n: np.ctypeslib.as_array((t * n).from_address(p)).copy()  # noqa: E731
        out = {"bits": d.bits, "k": k, "n": d.n, "s": arr(d.smooth_scales, C.c_double, k),
               "t_x": d.t_x, "e_x": arr(d.ext_x, C.c_int64, k), "block_x": d.block_x,
               "t_w": d.t_w, "e_w": arr(d.ext_w, C.c_int64, c1), "block_w": d.block_w,
               "act_scale": d.act_scale, "w_scale": d.w_scale, "kl_ratio_act": ka.value,
               "kl_ratio_w": kw.value}
        if d.weight_q:
            kp = -(-(c1 + int(out["e_w"].sum())) // d.block_w) * d.block_w
            out["weight_q"] = arr(d.weight_q, C.c_int32, kp * d.n).reshape(kp, d.n)
        return out

    def infer(self, input_path: str, out_path: str) -> tuple[int, int]:
        """-> (saturated elements, tensors run)."""
        sat, ran = C.c_int64(), C.c_int64()
        check(lib().fqg_model_infer(self._h, input_path.encode(), out_path.encode(),
                                    C.byref(sat), C.byref(ran)))
        return sat.value, ran.value


def run_layer(cfg: LayerQuantConfig, x, device: int = 0) -> tuple[np.ndarray, int]:
    """fq::run_layer(cfg, x, saturation_events) -> (y f64 [M, N], saturation)."""
    return Layer(cfg, device).run_layer(x)


def recipe_plan(weight, act_maxes, bits: int, alpha: float = 0.5, beta: float = 1.3,
                block: int = 32, smooth: bool = True, clip: bool = True) -> LayerQuantConfig:
    """Stages of fq::quantize_layer (pipeline.cpp:76-138) for a pinned bit width;
    the weight tail runs on the device when a :class:`Layer` is created."""
    w = _f64(weight)
    k, n = w.shape
    a = _f64(act_maxes)
    s = np.zeros(k)
    ex = np.zeros(k, np.int64)
    t_x, t_w, c1, kp, act = C.c_double(), C.c_double(), C.c_int64(), C.c_int64(), C.c_double()
    # plan_w has plan_x.padded_width entries: size for the common case, and
    # retry once with the exact width the call reports if that was too small.
    ew = np.zeros(4 * k + 64, np.int64)
    for attempt in range(2):
        rc = lib().fqg_recipe_plan(w.ctypes.data, k, n, a.ctypes.data, bits, alpha, beta, block,
                                   int(smooth), int(clip), s.ctypes.data, C.byref(t_x),
                                   ex.ctypes.data, C.byref(c1), C.byref(t_w), ew.ctypes.data,
                                   ew.shape[0], C.byref(kp), C.byref(act))
        if rc == _lib.ERR_INVALID and attempt == 0 and c1.value > ew.shape[0]:
            ew = np.zeros(c1.value, np.int64)
            continue
        check(rc)
        break
    px = FlattenPlan.from_extensions(t_x.value, ex, block)
    pw = FlattenPlan.from_extensions(t_w.value, ew[: c1.value], block)
    return LayerQuantConfig(bits=bits, smooth_scales=s, plan_x=px, plan_w=pw,
                            act_scale=act.value, weight=w)


def collect_channel_maxes(calib) -> np.ndarray:
    """fq::collect_channel_maxes (calibration.cpp:9-28) over [S, R, K] or [R, K]."""
    c = _f64(calib)
    c = c.reshape(-1, c.shape[-1])
    out = np.zeros(c.shape[1])
    lib().fqg_collect_channel_maxes(c.ctypes.data, c.shape[0], c.shape[1], out.ctypes.data)
    return out


def quantize_layer(weight, calib, bits: int, **kw) -> LayerQuantConfig:
    """fq::quantize_layer (pipeline.cpp:76-152), O1/O2 with the bit width pinned."""
    return recipe_plan(weight, collect_channel_maxes(calib), bits, **kw)


def synthetic_layer(index: int = 0, test_rows: Optional[int] = None, **kw):
    """fq::make_synthetic_layer (synthetic.cpp:121-159) ->
    (weight [K,N], calib [S,R,K], test_input [test_rows,K])."""
    o = _lib.SynthOpts()
    lib().fqg_synth_default(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    tr = o.rows if test_rows is None else test_rows
    w = np.zeros((o.in_channels, o.out_channels))
    calib = np.zeros((o.samples, o.rows, o.in_channels))
    x = np.zeros((tr, o.in_channels))
    check(lib().fqg_synthetic_layer(C.byref(o), index, w.ctypes.data, calib.ctypes.data,
                                    x.ctypes.data, tr))
    return w, calib, x
