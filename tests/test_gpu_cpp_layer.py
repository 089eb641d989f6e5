"""The MoE layer driven from C++ through the C-ABI alone (tests/cpp/
layer_plugin_demo.cpp): resident vs offloaded (shared slot pool, InfMoE
order) bit-identical, the order a permutation, every token routed, and the
measured timeline clean under infmoe_replay_check — no Python on the path."""
import subprocess
from pathlib import Path

import pytest

import paper_2106_10715_b200 as im

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def test_layer_from_cpp_through_the_c_abi(tmp_path):
    exe = tmp_path / "layer_plugin_demo"
    lib_dir = Path(im.library_path()).parent
    subprocess.run(["/usr/bin/g++", "-std=c++17", "-O2", str(ROOT / "tests" / "cpp" / "layer_plugin_demo.cpp"),
                    "-o", str(exe), f"-I{ROOT / 'include'}", "-I/usr/local/cuda/include",
                    f"-L{lib_dir}", "-linfmoe", f"-Wl,-rpath,{lib_dir}",
                    "-L/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64"],
                   check=True, capture_output=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "layer plugin demo ok" in r.stdout, r.stdout + r.stderr
