"""The C-ABI boundary: libfqg.so loads on a CPU-only host, exports every
function include/fqg.h declares, exposes only extern "C" names, and the Python
binding declares a signature for each; built for sm_100a only."""
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fqg.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fqg_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = header_functions()
    for required in ("fqg_layer_create", "fqg_layer_forward", "fqg_layer_run_host",
                     "fqg_layer_quantize_acts", "fqg_layer_gemm", "fqg_gemm",
                     "fqg_layer_quantize_acts_ex", "fqg_layer_gemm_ex",
                     "fqg_layer_destroy", "fqg_last_error", "fqg_build_flatten_plan"):
        assert required in names


def test_library_exports_every_declared_symbol(fq):
    from paper_2402_17985_b200 import _lib

    lib = fq.lib()
    missing = [n for n in header_functions() if not hasattr(lib, n)]
    assert not missing, f"not exported: {missing}"
    undeclared = [n for n in header_functions() if n not in _lib.SIGNATURES]
    assert not undeclared, f"no ctypes signature: {undeclared}"


def test_exports_are_plain_c(fq):
    from paper_2402_17985_b200 import _lib

    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    fqg = {l.split()[-1] for l in out.splitlines() if " T fqg_" in l}
    assert set(header_functions()) <= fqg


def test_sm100a_only_cubin(fq):
    from paper_2402_17985_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_tcgen05_and_tma_in_sass(fq):
    """The GEMM is tcgen05 (UTCIMMA incl. the CTA-pair form) fed by TMA."""
    from paper_2402_17985_b200 import _lib

    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True,
                          text=True).stdout
    for mnem in ("UTCIMMA", "UTCIMMA.2CTA", "UTMALDG.2D", "LDTM"):
        assert mnem in sass, mnem
    assert "HMMA" not in sass and "IMMA." not in sass.replace("UTCIMMA", "")


def test_error_codes_and_messages(fq):
    import ctypes as C

    import numpy as np

    e = np.zeros(1, np.int64)
    c, p = C.c_int64(), C.c_int64()
    rc = fq.lib().fqg_build_flatten_plan(np.array([1.0]).ctypes.data, 1, 0.0, 32, e.ctypes.data,
                                         None, C.byref(c), C.byref(p))
    assert rc == -2 and b"threshold" in fq.lib().fqg_last_error()
