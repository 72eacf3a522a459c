"""CPU checks of the boundary: libgpbo.so loads and exports every entry point include/gpbo.h
and include/gpbo_test.h (the test / diagnostic hooks) declare (no compute calls -- there is no
GPU here)."""
import ctypes
import os
import re

from paper_2403_08131_b200 import gpbo

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = "".join(open(os.path.join(ROOT, "include", h)).read() for h in ("gpbo.h", "gpbo_test.h"))
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*([a-z_0-9]+)\s*\(", src, re.M))


def test_library_exports_every_declared_symbol():
    lib = gpbo.load()
    names = declared_functions()
    assert {"gp_fit", "gp_posterior", "ei_score_argmax"} <= names
    for name in names:
        assert hasattr(lib, name), name
        assert ctypes.cast(getattr(lib, name), ctypes.c_void_p).value
    assert set(gpbo.exported_symbols()) == names


def test_version_and_argument_validation_without_gpu():
    assert "sm_100a" in gpbo.version()
    lib = gpbo.load()
    # null ctx / out pointers are rejected before any CUDA call
    assert lib.gpbo_ctx_create(0, None, 0, 0, None, None) == gpbo.EINVAL
    assert lib.gpbo_ctx_create(0, None, 2, 0, None, None) == gpbo.EINVAL
    assert lib.gp_fit(None, None, None, None, None) == gpbo.EINVAL
    assert lib.ei_score_argmax(None, None, None, None, None, None, 0, None, None) == gpbo.EINVAL


def test_no_oracle_import_in_product_package():
    pkg = os.path.join(ROOT, "paper_2403_08131_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
