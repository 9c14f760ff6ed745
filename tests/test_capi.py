"""The C-ABI library loads without a GPU and exports every symbol
include/dfa2c.h declares (no compute calls here)."""
import os
import re
import subprocess

from paper_2503_22796_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "dfa2c.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dfa2c_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    names = declared_symbols()
    assert len(names) >= 25
    for n in names:
        assert hasattr(L, n), n
    nm = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in nm.splitlines() if line.strip()}
    assert set(names) <= exported
    # every declared entry point has a ctypes signature in the binding
    assert set(names) == set(_lib.exported_symbols())


def test_version_and_error_channel():
    L = _lib.lib()
    assert b"sm_100a" in L.dfa2c_version()
    d = _lib.Dims(0, 64, 10, 0, 0)
    import ctypes
    rc = L.dfa2c_arrow_mask(ctypes.byref(d), 8, 0, None, None)
    assert rc == 1 and b"n_heads" in L.dfa2c_last_error()


def test_library_contains_sm100a_tcgen05_and_tma_code():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "attn_fwd_sm100" in out
    assert "UTCHMMA" in out or "UTCQMMA" in out or "UTCMMA" in out  # tcgen05.mma
    assert "UTMALDG" in out                                        # TMA loads
    assert "LDTM" in out and "STTM" in out                          # TMEM ld / st
    assert "HMMA" not in out.replace("UTCHMMA", "")                 # no legacy mma.sync path
