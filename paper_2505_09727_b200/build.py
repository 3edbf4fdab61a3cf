"""Build recipe for libesp_b200.so (sm_100a), in-tree.

    python paper_2505_09727_b200/build.py           # incremental
    python paper_2505_09727_b200/build.py --force   # rebuild everything

(run by path: importing the package itself requires the built library)

nvcc cross-compiles for `-gencode arch=compute_100a,code=sm_100a` without a
GPU, so this runs in the CPU container; the resulting .so travels to the
GPU box with the repo snapshot.  Objects are cached next to the sources
(build/ is git-ignored) and rebuilt when a source or header is newer.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "esp_b200")
LIB = os.path.join(PKG, "libesp_b200.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-pthread",
          "-I" + os.path.join(ROOT, "include")]
SOURCES = ["plan.cpp", "plan_device.cu", "engine.cu", "direct.cu", "capi.cpp", "shard.cu"]
HEADERS = ["plan.hpp", "engine.hpp", "direct.hpp", "capi_internal.hpp", os.path.join("..", "..", "include", "esp_b200.h")]


def _newest_header() -> float:
    return max(os.path.getmtime(os.path.join(CSRC, h)) for h in HEADERS)


VARIANT = None   # experiments: --variant NAME -DX=Y ... -> libesp_b200_NAME.so (ESP_B200_LIB loads it)
DEFINES: list = []


def _paths(checked: bool):
    """(object directory, library) of the product or the checked build."""
    if VARIANT:
        return BUILD + "_" + VARIANT, os.path.join(PKG, f"libesp_b200_{VARIANT}.so")
    if checked:
        return BUILD + "_checked", os.path.join(PKG, "libesp_b200_checked.so")
    return BUILD, LIB


def _compile(src: str, checked: bool = False) -> str:
    path = os.path.join(CSRC, src)
    obj = os.path.join(_paths(checked)[0], src + ".o")
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(path),
                                                            _newest_header()):
        return obj
    cmd = [NVCC, *ARCH, *COMMON, *DEFINES, "-c", path, "-o", obj]
    if checked:
        cmd += ["-DESP_DEVICE_CHECKS"]
    if src.endswith(".cu"):
        cmd += ["-Xptxas", "-warn-spills"]
    else:
        cmd += ["-x", "cu"] if src == "capi.cpp" else []
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip():
        sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False, verbose: bool = True, checked: bool = False) -> str:
    """Compile libesp_b200.so (or, checked=True, libesp_b200_checked.so with
    the device-side bounds checks ESP_DCHECK compiled in, loaded by the
    package when ESP_B200_CHECKED=1)."""
    bdir, LIB = _paths(checked)
    os.makedirs(bdir, exist_ok=True)
    if force:
        for s in SOURCES:
            o = os.path.join(bdir, s + ".o")
            if os.path.exists(o):
                os.remove(o)
    with ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(lambda src: _compile(src, checked), SOURCES))
    if (not os.path.exists(LIB)) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcufft", "-cudart", "static",
               "-Xlinker", "-rpath=" + os.path.join(CUDA, "lib64"), "-Xcompiler", "-pthread", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        if verbose:
            print(f"built {LIB}")
    return LIB


if __name__ == "__main__":
    if "--variant" in sys.argv:
        VARIANT = sys.argv[sys.argv.index("--variant") + 1]
        DEFINES = [a for a in sys.argv if a.startswith("-D")]
    build(force="--force" in sys.argv, checked="--checked" in sys.argv)
