"""Host-side checks of the C-ABI library (no GPU needed, `-m "not gpu"`).

The library must load and export every symbol include/geninv.h declares;
the binding must declare the same names; without a GPU the binding must
refuse to run (there is no CPU fallback).
"""
import ctypes
import os
import re

import pytest
import torch

from paper_0804_4809_b200 import binding, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "geninv.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"GENINV_API\s+[\w\s\*]+?\b(geninv_\w+)\s*\(", txt)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for need in ["geninv_d", "geninv_host_d", "geninv_batched_d", "geninv_gram_d", "geninv_from_gram_d",
                 "geninv_apply_d", "geninv_frchol_d", "geninv_spd_inverse_d", "geninv_create", "geninv_destroy"]:
        assert need in syms


def test_library_builds_and_exports_every_declared_symbol():
    lib_path = build.build()
    lib = ctypes.CDLL(lib_path)
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_binding_covers_the_header():
    assert sorted(binding.EXPORTED) == declared_symbols()


def test_strerror_without_gpu():
    lib = binding.load()
    lib.geninv_strerror.restype = ctypes.c_char_p
    assert lib.geninv_strerror(0) == b"ok"
    assert b"SPD" in lib.geninv_strerror(3)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    with pytest.raises(RuntimeError):
        binding.Handle()


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_0804_4809_b200")
    bad = re.compile(r"^\s*(from\s+oracle|import\s+oracle|#\s*include\s*[<\"].*oracle)|geninv_oracle|import_module\(.oracle",
                     re.M)
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                assert not bad.search(open(os.path.join(dirpath, f)).read()), f
