#!/usr/bin/env python3
"""Generates tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref,
built from /root/reference/proj/core by oracle/Makefile). Run in a container
that has /root/reference; the fixtures are committed so the tests (and the GPU
box, which has no /root/reference) never need the reference itself.

Each fixture: the reference synthetic layer (fq::make_synthetic_layer, seed 42),
the recipe of fq::quantize_layer (O1 -> 8 bits, O2 with gamma=1e6 -> 4 bits),
and the outputs of the activation half of fq::run_layer (quantized operand,
saturation count), fq::int_matmul_raw (int64 accumulators) and fq::run_layer
(f64 outputs) on the held-out test input, plus the same on a 3x-scaled input
that saturates.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import Ref  # noqa: E402

CONFIGS = [
    # name, K, N, rows, samples, index, mode, gamma
    ("ref128_o1", 128, 128, 32, 8, 0, 1, 1.86),   # the reference's default model size
    ("ref128_o2", 128, 128, 32, 8, 1, 2, 1e6),
    ("k256_n96_o1", 256, 96, 24, 4, 2, 1, 1.86),
    ("k192_n160_o2", 192, 160, 40, 3, 3, 2, 1e6),
]


def main():
    ref = Ref()
    for name, k, n, rows, samples, index, mode, gamma in CONFIGS:
        w, calib, x, outl = ref.synthetic_layer(index, in_channels=k, out_channels=n, rows=rows,
                                                samples=samples)
        rl = ref.quantize_layer(w, calib, mode=mode, gamma=gamma)
        L = rl.to_layer()
        out = dict(weight=w, calib=calib, x=x, outliers=outl, bits=L.bits, s=L.s, t_x=L.t_x,
                   e_x=L.e_x, t_w=L.t_w, e_w=L.e_w, act_scale=L.act_scale, s_w=L.s_w,
                   wq=L.wq.astype(np.int8))
        for tag, xi in (("", x), ("_sat", x * 3.0)):
            qx, sat = rl.quantized_acts(xi)
            acc = ref.int_matmul_raw(qx, L.wq, L.bits, L.bits)
            y, sat2 = rl.run_layer(xi)
            assert sat == sat2
            out["qx" + tag] = qx.astype(np.int8)
            out["acc" + tag] = acc.astype(np.int32)
            assert np.array_equal(out["acc" + tag].astype(np.int64), acc)
            out["y" + tag] = y
            out["sat" + tag] = sat
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **out)
        print(f"{name}: K={k} N={n} bits={L.bits} C1={L.c1} K'={L.kp} sat={out['sat']}/"
              f"{out['sat_sat']} -> {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
