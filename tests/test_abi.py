"""CPU-side checks of the C-ABI library: it builds for sm_100a, loads, and
exports every symbol include/bte.h declares; the binding refuses to run
without a GPU (no CPU fallback).  No compute calls here."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bte.h")


def _declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"BTE_API\s+[\w\s\*]*?\b(bte_\w+)\s*\(", txt)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2305_19400_b200 import build
    return build.build()


def test_header_declares_entry_points():
    names = _declared()
    for n in ("bte_create", "bte_set_bc", "bte_step", "bte_get_intensity", "bte_get_temperature",
              "bte_destroy", "bte_last_error", "bte_set_state"):
        assert n in names


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    for n in _declared():
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (bte_\w+)", out))
    assert exported == set(_declared())
    lib.bte_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.bte_version()


def test_library_is_sm100a(libpath):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_binding_has_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import bte_inputs as bi
    from paper_2305_19400_b200 import Solver
    with pytest.raises(RuntimeError):
        Solver.from_problem(bi.small_3d())


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2305_19400_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "bte_oracle" not in txt, f
