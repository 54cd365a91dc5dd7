"""CPU: the C-ABI library is built for sm_100a, loads without a GPU and
exports every symbol include/gift_b200.h declares; the product package
never touches the oracle and fails loudly without a device."""

from __future__ import annotations

import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gift_b200.h")
PKG = os.path.join(ROOT, "paper_2502_17632_b200")


def header_functions() -> set[str]:
    src = open(HEADER).read()
    return set(re.findall(r"^\s*(?:const\s+)?[\w\*\s]+?\b(gift_\w+)\s*\(", src, flags=re.M))


@pytest.fixture(scope="module")
def lib():
    from paper_2502_17632_b200 import _lib, build_ext

    build_ext.build()
    return _lib.load_library()


def test_header_declares_the_api():
    names = header_functions()
    for must in ("gift_build_clique_graph", "gift_csr_from_coo", "gift_filter", "gift_filter_host",
                 "gift_place_host", "gift_normalized_augmented_adjacency", "gift_csr_matmul", "gift_csr_degrees"):
        assert must in names


def test_every_declared_symbol_is_exported(lib):
    missing = [n for n in sorted(header_functions()) if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_table_matches_header():
    from paper_2502_17632_b200 import _lib

    assert {n for n, _, _ in _lib.SIGNATURES} == header_functions()


def test_version_string_without_device(lib):
    assert b"sm_100a" in lib.gift_version()


def test_library_is_sm100a_cubin(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", os.path.join(PKG, "libgiftb200.so")],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_product_never_imports_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "from oracle" not in src and "import oracle" not in src, f
                assert "gift_oracle" not in src, f


def test_no_device_means_loud_failure():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a device is visible")
    import numpy as np

    import paper_2502_17632_b200 as gb

    fd = gb.FlatDesign(np.array([0, 2]), np.array([0, 1]), np.zeros(2, bool), np.full((2, 2), np.nan),
                       gb.Region(0, 0, 1, 1))
    with pytest.raises(gb.DeviceError):
        gb.build_clique_graph(fd)
    with pytest.raises(gb.DeviceError):
        gb.from_coo(2, [0, 1], [1, 0], [1.0, 1.0])
