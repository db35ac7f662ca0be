"""CPU checks of the boundary: libgx.so loads without a GPU and exports every function that
include/gx.h declares; the Python binding exposes the same names; the CUDA path fails loudly
(no CPU fallback) when there is no device."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    text = open(os.path.join(ROOT, "include", "gx.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gx_\w+)\s*\(", text)))


def test_header_declares_the_north_star_calls():
    names = declared()
    for required in ("gx_load_prog", "gx_verify", "gx_create_map", "gx_run_batch", "gx_read_map"):
        assert required in names


def test_library_exports_every_declared_symbol():
    import paper_2512_12615_b200 as gx
    L = gx.lib()
    missing = [n for n in declared() if not hasattr(L, n)]
    assert not missing, missing


def test_binding_has_same_names():
    import paper_2512_12615_b200 as gx
    for n in declared():
        assert hasattr(gx, n), n
        assert n in gx.EXPORTS, n


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2512_12615_b200 as gx
    with pytest.raises(gx.GxError):
        gx.Runtime(0)


def test_product_does_not_import_oracle():
    """The product path never imports, links or executes anything under oracle/."""
    pkg = os.path.join(ROOT, "paper_2512_12615_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".h", ".cuh")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*|/\*.*?\*/|\"\"\".*?\"\"\"", "", src, flags=re.S).lower() \
                    or f == "__init__.py" and "import oracle" not in src, f
