"""§8f row 2: the reference's on-disk contract -> device layers.

The UNMODIFIED reference (oracle/_ref: fq_core + schemas.cpp + archive.cpp)
writes a recipe JSON and an FQTA quantized archive exactly as its CLI's
cmd_quantize does (flattenquant_cli.cpp:199-238); fqg_model_load parses them
(CPU tests: every recipe field equals the reference's in-memory config) and
builds device layers whose cmd_infer output archive is byte-identical to the
reference cmd_infer's (GPU test).
"""
import json
import os

import numpy as np
import pytest

LAYERS = [("blk0.qkv", 0, 256, 192, 2), ("blk0.o", 1, 192, 256, 1), ("blk1.fc", 2, 256, 320, 2)]


def write_reference_model(ref, tmp_path):
    rls, names, inputs = [], [], {}
    for name, idx, k, n, mode in LAYERS:
        w, calib, x, _ = ref.synthetic_layer(idx, in_channels=k, out_channels=n, rows=32,
                                             samples=4)
        rls.append(ref.quantize_layer(w, calib, mode=mode, gamma=1e6 if mode == 2 else 1.86))
        names.append(name)
        inputs[f"{name}/x"] = x
        inputs[f"{name}/x3"] = x * 3.0  # saturating rows
    recipe, qmodel, inp = (str(tmp_path / f) for f in ("recipe.json", "model.fqta", "in.fqta"))
    ref.write_model(rls, names, recipe, qmodel)
    ref.write_f64_archive(inp, inputs)
    return rls, names, recipe, qmodel, inp


def test_recipe_and_archive_parse_like_the_reference(ref, fq, tmp_path):
    rls, names, recipe, qmodel, _ = write_reference_model(ref, tmp_path)
    m = fq.Model(recipe, qmodel, device=-1)
    assert m.names == names
    for i, rl in enumerate(rls):
        L = rl.to_layer()
        r = m.recipe(i)
        assert r["bits"] == L.bits and r["k"] == L.k and r["n"] == L.n
        assert np.array_equal(r["s"], L.s)  # "%.17g" strings round-trip exactly
        assert r["t_x"] == L.t_x and r["t_w"] == L.t_w
        assert np.array_equal(r["e_x"], L.e_x) and np.array_equal(r["e_w"], L.e_w)
        assert r["act_scale"] == L.act_scale and r["w_scale"] == L.s_w
        assert np.array_equal(r["weight_q"], L.wq)
        assert r["kl_ratio_act"] == rl.info.kl_ratio_act


def test_recipe_errors_are_the_reference_errors(ref, fq, tmp_path):
    _, _, recipe, qmodel, _ = write_reference_model(ref, tmp_path)
    doc = json.load(open(recipe))
    doc["layers"][0]["plan_x"]["c_extend"] += 1
    bad = str(tmp_path / "bad.json")
    json.dump(doc, open(bad, "w"))
    with pytest.raises(fq.FqgInvalidArgument, match="plan: inconsistent extension counts"):
        fq.Model(bad, qmodel, device=-1)
    doc = json.load(open(recipe))
    doc["schema_version"] = 2
    json.dump(doc, open(bad, "w"))
    with pytest.raises(fq.FqgInvalidArgument, match="unsupported schema_version 2"):
        fq.Model(bad, qmodel, device=-1)
    doc = json.load(open(recipe))
    doc["layers"][1]["layer"] = "renamed"
    json.dump(doc, open(bad, "w"))
    with pytest.raises(fq.FqgRuntimeError, match="missing tensor: renamed.qweight"):
        fq.Model(bad, qmodel, device=-1)
    raw = open(qmodel, "rb").read()
    trunc = str(tmp_path / "trunc.fqta")
    open(trunc, "wb").write(raw[:-7])
    with pytest.raises(fq.FqgRuntimeError, match="truncated payload"):
        fq.Model(recipe, trunc, device=-1)
    open(trunc, "wb").write(b"NOPE" + raw[4:])
    with pytest.raises(fq.FqgRuntimeError, match="bad magic"):
        fq.Model(recipe, trunc, device=-1)


@pytest.mark.gpu
@pytest.mark.parametrize("a_fmt", ["i8", "i4"])
def test_infer_archive_is_byte_identical_to_reference_cmd_infer(ref, fq, tmp_path, a_fmt):
    _, _, recipe, qmodel, inp = write_reference_model(ref, tmp_path)
    out_ref, out_gpu = str(tmp_path / "out_ref.fqta"), str(tmp_path / "out_gpu.fqta")
    sat_ref, ran_ref = ref.infer(qmodel, recipe, inp, out_ref)
    m = fq.Model(recipe, qmodel, device=0, a_format=fq.I8 if a_fmt == "i8" else fq.I4)
    sat, ran = m.infer(inp, out_gpu)
    assert (sat, ran) == (sat_ref, ran_ref) and sat_ref > 0
    assert open(out_gpu, "rb").read() == open(out_ref, "rb").read()
    assert os.path.getsize(out_gpu) > 0
