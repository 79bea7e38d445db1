"""CPU checks of the C ABI: the library loads without a GPU and exports
exactly the symbols include/zo_b200.h declares (no compute calls here)."""

import os
import re

import pytest

from paper_2507_03211_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "zo_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(zo_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert _declared() == sorted(L.SIGNATURES)


def test_library_loads_and_exports_every_symbol():
    if not os.path.exists(L.LIB_PATH):
        pytest.skip("library not built")
    dll = L.load()
    for name in _declared():
        assert hasattr(dll, name), name
    assert dll.zo_version().decode().startswith("zo_b200")
    assert dll.zo_perturb_tile_elems() == 512
    assert dll.zo_gemm_ce_tiles(50272) == 394


def test_sass_is_sm100a_tcgen05():
    import shutil
    import subprocess

    if not os.path.exists(L.LIB_PATH) or not shutil.which("cuobjdump"):
        pytest.skip("library or cuobjdump missing")
    sass = subprocess.run(["cuobjdump", "-sass", L.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", L.LIB_PATH], capture_output=True, text=True).stdout
    for mnemonic in ("UTCHMMA", "UTMALDG", "LDTM"):
        assert mnemonic in sass, mnemonic
