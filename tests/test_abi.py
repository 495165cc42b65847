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


def test_fused_readout_rejects_bad_arguments_before_any_device_work():
    """dgc_readout_f16 / _evolve validate their arguments on the host (error
    code + dgc_last_error message, no CUDA call): H must be 128, C 16 or 32,
    n positive, the outputs 16-byte aligned."""
    from paper_2309_03523_b200 import _native
    lib = _native.lib()
    base = [None, None, None, None]
    cases = [
        ("dgc_readout_f16", (100, 64, 16), "H must be 128"),
        ("dgc_readout_f16", (100, 128, 8), "C must be 16 or 32"),
        ("dgc_readout_f16", (0, 128, 16), "bad row count"),
        ("dgc_readout_f16_evolve", (100, 128, 24), "C must be 16 or 32"),
    ]
    for name, (n, H, C), msg in cases:
        fn = getattr(lib, name)
        tail = [None] * (5 if name == "dgc_readout_f16" else 6)
        rc = fn(*base, n, H, C, 1.0, 1.0, *tail)
        assert rc != 0, name
        err = lib.dgc_last_error().decode()
        assert msg in err, (name, err)
    # misaligned output pointer (never dereferenced: the check comes first)
    rc = lib.dgc_readout_f16(None, None, None, None, 100, 128, 16, 1.0, 1.0, 8, None, None, 16, None)
    assert rc != 0 and "16-byte aligned" in lib.dgc_last_error().decode()
