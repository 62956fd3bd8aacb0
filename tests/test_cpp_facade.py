"""include/gempe.hpp: reference-style C++ (namespace entropy_embed = gempe) compiles and links against the
library; on a GPU box the program also runs."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "facade_test.cpp")


def _build(tmp_path):
    from paper_2011_03479_b200 import _capi
    _capi.load()
    lib_dir = os.path.dirname(_capi.library_path())
    exe = str(tmp_path / "facade_test")
    subprocess.check_call(["g++", "-std=c++17", "-O1", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"), SRC, "-o", exe,
                           "-L", lib_dir, "-lgempe_b200", f"-Wl,-rpath,{lib_dir}"])
    return exe


def test_reference_style_cpp_compiles_and_links(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_reference_style_cpp_runs(tmp_path):
    out = subprocess.run([_build(tmp_path)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "facade_test: OK" in out.stdout
