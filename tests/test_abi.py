"""The C-ABI library loads and exports every symbol include/capt_b200.h
declares (CPU only: no compute calls)."""

import ctypes
import os
import re

from conftest import ROOT


def _declared():
    src = open(os.path.join(ROOT, "include", "capt_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(capt_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_entry_points():
    names = _declared()
    for must in ("capt_tree_create", "capt_tree_build", "capt_query", "capt_leaf_indices",
                 "capt_filter_cloud", "capt_tree_export", "capt_tree_destroy",
                 "capt_last_error"):
        assert must in names


def test_library_exports_all_declared_symbols():
    from paper_2406_02807_b200 import _lib
    L = ctypes.CDLL(_lib.lib()._name)
    missing = [n for n in _declared() if not hasattr(L, n)]
    assert not missing, missing
    assert set(_lib.EXPORTED_SYMBOLS) == set(_declared())
    assert L.capt_version() == 1


def test_library_is_sm100a():
    from paper_2406_02807_b200 import _lib
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True)
    assert "sm_100a" in out.stdout
