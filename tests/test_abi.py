"""The C-ABI library loads and exports every symbol include/dgc_b200.h
declares (no compute calls: runs without a GPU)."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared():
    text = (ROOT / "include" / "dgc_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:[\w\*\s]+?)\b(dgc_\w+)\(", text, flags=re.M)))


def test_header_declares_entry_points():
    names = declared()
    assert "dgc_gemm_tf32" in names and "dgc_spmm_csr" in names and "dgc_rnn_fwd" in names
    assert len(names) >= 20


def test_library_exports_all_declared_symbols():
    from paper_2309_03523_b200 import _native
    lib = _native.lib()
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(declared()) == set(_native.exported_symbols())
    assert lib.dgc_version() == 1


def test_library_is_sm100a():
    import subprocess
    from paper_2309_03523_b200 import _native
    out = subprocess.run(["cuobjdump", "--list-elf", str(_native.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", str(_native.LIB_PATH)], capture_output=True,
                          text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass
