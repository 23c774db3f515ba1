"""The C-ABI library builds, loads without a GPU, and exports every symbol
include/fzb200.h declares (no compute calls here)."""

import ctypes
import os
import re

from conftest import ROOT


def _declared():
    src = open(os.path.join(ROOT, "include", "fzb200.h")).read()
    return sorted(set(re.findall(r"FZB_API\s+[\w\s\*]+?\b(fzb_\w+)\s*\(", src)))


def test_header_declares_entry_points():
    names = _declared()
    assert "fzb_lorenzo_encode_f32" in names and "fzb_huffman_decode" in names
    assert len(names) >= 20


def test_library_exports_every_declared_symbol():
    from paper_2509_20563_b200 import _lib
    L = _lib.load()
    for name in _declared():
        assert hasattr(L, name), name
    assert set(_declared()) == set(_lib.EXPORTED)
    assert L.fzb_abi_version() == 1


def test_workspace_queries_are_host_only():
    from paper_2509_20563_b200 import _lib
    L = _lib.load()
    assert L.fzb_lorenzo_workspace_bytes(512, 512, 512) > 0
    assert L.fzb_lorenzo_workspace_bytes(1, 1, 280953867) > 0
    assert L.fzb_huffman_build_workspace_bytes(1024) > 0
    assert L.fzb_bitshuffle_workspace_bytes(1 << 27) > 0
