"""Build libinfmoe.so in-tree (paper_2106_10715_b200/_lib/) for sm_100a.

nvcc cross-compiles the CUDA translation units (no GPU needed), g++ the host
planner; everything links into one C-ABI shared library whose exports are
declared in include/infmoe.h.  Usage: python paper_2106_10715_b200/build.py
(not `-m`: importing the package requires the library this script builds).
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_lib"
OBJ_DIR = ROOT / "build" / "obj"
LIB = OUT_DIR / "libinfmoe.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
HOST_CXX = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
INCLUDES = [f"-I{ROOT / 'include'}", f"-I{CSRC}"]

CU_SOURCES = [
    "kernels/fill.cu",
    "kernels/gate.cu",
    "kernels/dispatch.cu",
    "kernels/expert_gemm.cu",
    "kernels/ep_peer.cu",
    "kernels/codec.cu",
    "runtime/layer.cu",
    "runtime/capi_device.cu",
]
CXX_SOURCES = [
    "host/planner.cpp",
    "host/capi_host.cpp",
    "host/ep_plan.cpp",
    "host/scenario.cpp",
    "runtime/nccl_shim.cpp",
    "runtime/scenario_run.cpp",
    "runtime/capi_scenario.cpp",
]
CLI = OUT_DIR / "infmoe"


def _json_include() -> str:
    """nlohmann json 3.11.3 (header-only; compile time only): the copy the image
    ships with cudnn_frontend, the same release the reference vendors."""
    import sysconfig
    cands = [Path(sysconfig.get_paths()["purelib"]) / "include" / "cudnn_frontend" /
             "thirdparty" / "nlohmann",
             Path("/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/"
                  "thirdparty/nlohmann")]
    for c in cands:
        if (c / "json.hpp").exists():
            return str(c)
    raise RuntimeError("json.hpp (nlohmann 3.11.3) not found")


def _headers_digest() -> str:
    h = hashlib.sha256()
    for p in sorted(list(CSRC.rglob("*.hpp")) + list(CSRC.rglob("*.cuh")) +
                    [ROOT / "include" / "infmoe.h"]):
        h.update(p.read_bytes())
    return h.hexdigest()[:16]


def _compile(src: str, digest: str, verbose: bool) -> Path:
    path = CSRC / src
    obj = OBJ_DIR / (src.replace("/", "_") + ".o")
    stamp = obj.with_suffix(".stamp")
    key = hashlib.sha256(path.read_bytes() + digest.encode()).hexdigest()
    if obj.exists() and stamp.exists() and stamp.read_text() == key:
        return obj
    if src.endswith(".cu"):
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++20", "-ccbin", HOST_CXX,
               "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3",
               "--expt-relaxed-constexpr", *INCLUDES, "-c", str(path), "-o", str(obj)]
    else:
        cmd = [HOST_CXX, "-O2", "-std=c++20", "-fPIC", "-Wall", "-ffp-contract=off",
               *INCLUDES, f"-I/usr/local/cuda/include", f"-I{_json_include()}", "-c", str(path),
               "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {src}\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    stamp.write_text(key)
    return obj


def build(verbose: bool = False) -> Path:
    OBJ_DIR.mkdir(parents=True, exist_ok=True)
    OUT_DIR.mkdir(parents=True, exist_ok=True)
    digest = _headers_digest()
    srcs = CU_SOURCES + CXX_SOURCES
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, digest, verbose), srcs))
    # relink whenever the set of object contents changed (content keys, not
    # mtimes: a copied-in or restored library must not be mistaken for fresh)
    link_key = hashlib.sha256("".join(o.with_suffix(".stamp").read_text() for o in objs)
                              .encode()).hexdigest()
    link_stamp = OBJ_DIR / "libinfmoe.stamp"
    if LIB.exists() and link_stamp.exists() and link_stamp.read_text() == link_key:
        _build_cli(link_key)
        return LIB
    cmd = [NVCC, *ARCH, "-shared", "-ccbin", HOST_CXX, "-o", str(LIB), *map(str, objs),
           "-lcudart", "-ldl", "-Xlinker", "-rpath,/usr/local/cuda/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    link_stamp.write_text(link_key)
    _build_cli(link_key)
    return LIB


def _build_cli(link_key: str) -> None:
    """The scenario CLI (`infmoe run|sweep|resolve`), a thin C++ front end over
    libinfmoe.so (loaded from its own directory)."""
    src = CSRC / "cli" / "infmoe_cli.cpp"
    key = hashlib.sha256(src.read_bytes() + link_key.encode()).hexdigest()
    stamp = OBJ_DIR / "infmoe_cli.stamp"
    if CLI.exists() and stamp.exists() and stamp.read_text() == key:
        return
    cmd = [HOST_CXX, "-O2", "-std=c++20", "-Wall", *INCLUDES, str(src), "-o", str(CLI),
           f"-L{OUT_DIR}", "-linfmoe", "-Wl,-rpath,$ORIGIN"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"cli build failed\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    stamp.write_text(key)


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
