"""The C++ drop-in header (include/infmoe/moesim.hpp): a moesim-API program
(tests/cpp/test_moesim_compat.cpp) builds against it and libinfmoe.so, passes
the SPEC examples, and prints the same digest as the same program built
against the reference headers."""
import subprocess
from pathlib import Path

import pytest

import paper_2106_10715_b200 as im

ROOT = Path(__file__).resolve().parent.parent
SRC = ROOT / "tests" / "cpp" / "test_moesim_compat.cpp"
REF_INC = Path("/root/reference/proj/include")


def _build_and_run(tmp_path, use_infmoe: bool) -> str:
    exe = tmp_path / ("compat_infmoe" if use_infmoe else "compat_ref")
    lib_dir = Path(im.library_path()).parent
    cmd = ["/usr/bin/g++", "-std=c++20", "-O2", "-ffp-contract=off", str(SRC), "-o", str(exe)]
    if use_infmoe:
        cmd += ["-DUSE_INFMOE", f"-I{ROOT / 'include'}", f"-L{lib_dir}", "-linfmoe",
                f"-Wl,-rpath,{lib_dir}"]
    else:
        cmd += [f"-I{REF_INC}"]
    subprocess.run(cmd, check=True, capture_output=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    return r.stdout.strip()


def test_compat_header_passes_spec_examples(tmp_path):
    out = _build_and_run(tmp_path, True)
    assert out.endswith("failures 0")


@pytest.mark.skipif(not REF_INC.exists(), reason="reference headers not present")
def test_compat_header_matches_reference_build(tmp_path):
    assert _build_and_run(tmp_path, True) == _build_and_run(tmp_path, False)
