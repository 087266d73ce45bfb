"""In-tree build of the sm_100a extension (nvcc, no torch JIT cache).

The resulting ``_lcp_b200.so`` lives next to this file so it travels with the
repository snapshot to the GPU box.  cudart is linked statically, so the
library loads (and exports its C ABI) on hosts without a GPU driver.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
OUT = os.path.join(HERE, "_lcp_b200.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-shared", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
    "-cudart", "static",
]


def _sources() -> list[str]:
    files = glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
    files.append(os.path.join(ROOT, "include", "lcp_b200.h"))
    return files


def needs_build() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    return any(os.path.getmtime(f) > t for f in _sources())


HOST_SRC = os.path.join(CSRC, "host_submit.c")
HOST_OUT = os.path.join(HERE, "_lcp_host" + (sysconfig.get_config_var("EXT_SUFFIX") or ".so"))


def build_host(force: bool = False, verbose: bool = False) -> str:
    """The CPython fast path for async submissions (csrc/host_submit.c)."""
    if not force and os.path.exists(HOST_OUT) and os.path.getmtime(HOST_OUT) >= os.path.getmtime(HOST_SRC):
        return HOST_OUT
    cc = os.environ.get("CC", "gcc")
    tmp = HOST_OUT + ".tmp"
    cmd = [cc, "-O2", "-shared", "-fPIC", "-std=c11", "-Wall", "-Wextra",
           "-I", sysconfig.get_paths()["include"], "-o", tmp, HOST_SRC]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(tmp, HOST_OUT)
    return HOST_OUT


def build_native(force: bool = False, verbose: bool = False) -> str:
    build_host(force, verbose)
    if not force and not needs_build():
        return OUT
    nvcc = os.environ.get("NVCC", "nvcc")
    tmp = OUT + ".tmp"
    cmd = [nvcc, *NVCC_FLAGS, "-o", tmp, os.path.join(CSRC, "lcp_b200.cu")]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build_native(force=True, verbose=True))
