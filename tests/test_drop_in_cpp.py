"""Runs tests/cpp/test_drop_in: the unmodified reference C++ API (fq::quantize_layer,
fq::run_layer) next to the drop-in fq::gpu::run_layer, bit-exact on the GPU."""
import os
import subprocess

import pytest

BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "build", "test_drop_in")


@pytest.mark.gpu
def test_cpp_drop_in_matches_reference():
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/build/test_drop_in not built (needs /root/reference headers)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "ALL PASS" in r.stdout


def test_cpp_drop_in_fails_loudly_without_gpu():
    """Without a device the drop-in throws (std::runtime_error), never falls back."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    if not os.path.exists(BIN):
        pytest.skip("not built")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=120)
    assert r.returncode != 0 and "runtime_error" in r.stderr
