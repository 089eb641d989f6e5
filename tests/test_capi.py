"""The drop-in boundary: libinfmoe.so loads without a GPU and exports every
entry point include/infmoe.h declares (no compute calls here)."""
import re
import subprocess
from pathlib import Path

import paper_2106_10715_b200 as im

ROOT = Path(__file__).resolve().parent.parent


def _declared():
    text = (ROOT / "include" / "infmoe.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(infmoe_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    out = subprocess.run(["nm", "-D", "--defined-only", im.library_path()], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (infmoe_[a-z0-9_]+)", out))
    declared = _declared()
    assert len(declared) >= 30
    missing = [s for s in declared if s not in exported]
    assert not missing, missing


def test_library_is_sm100a_and_has_tcgen05():
    out = subprocess.run(["cuobjdump", "--list-elf", im.library_path()], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", im.library_path()], capture_output=True,
                          text=True).stdout
    for mnemonic in ("UTCHMMA", "UTMALDG", "LDTM"):
        assert mnemonic in sass, mnemonic


def test_no_cxx_exception_crosses_the_abi():
    # every failure is a status code + message, even for NULL arguments
    import ctypes as C
    lib = im._lib
    assert lib.infmoe_resident_capacity(None, None, None) == 6
    assert b"NULL" in lib.infmoe_last_error()
    assert lib.infmoe_schedule(None, 3, 1.0, 1, 0, 12, None, None, None) == 6
    assert lib.infmoe_layer_create(None, None) == 6
    assert lib.infmoe_layer_destroy(None) == 0
    assert im.version().startswith("infmoe-b200")
