"""The C-ABI library loads without a GPU and exports exactly what include/gempe.h declares."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "gempe.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gempe_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_list_agree():
    from paper_2011_03479_b200 import _capi
    assert declared_symbols() == sorted(_capi.SYMBOLS)


def test_library_exports_every_declared_symbol():
    from paper_2011_03479_b200 import _capi
    lib = _capi.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _capi.library_path()], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert set(declared_symbols()) <= exported
    # no torch / python types leak through the boundary, and nothing from the oracle is linked in
    assert not any("go_" == s[:3] or s.startswith("ref_") for s in exported)


def test_no_cpu_fallback_without_a_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2011_03479_b200 as P
    with pytest.raises(P.CudaError):
        P.Context(P.Graph(3, [0], [1]), 2)
    with pytest.raises(P.CudaError):
        P.embed(P.Graph(3, [0], [1]), 2)


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2011_03479_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".cuh", ".hpp", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "gempe_oracle" not in text and "libgempe_ref" not in text, f
