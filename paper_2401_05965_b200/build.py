"""Build the executor's CUDA library in-tree: paper_2401_05965_b200/libhap_b200.so.

    python -m paper_2401_05965_b200.build          # incremental
    python -m paper_2401_05965_b200.build --force

sm_100a only (tcgen05 / TMEM / TMA).  Objects are compiled in parallel into
build/ and linked against the NCCL the PyTorch wheel ships (same libnccl.so.2
the process already loads), with an rpath so the GPU box finds it.
"""
from __future__ import annotations

import argparse
import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libhap_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def nccl_paths() -> tuple[str, str]:
    import importlib.util

    spec = importlib.util.find_spec("nvidia")
    for base in list(spec.submodule_search_locations or []):
        inc = os.path.join(base, "nccl", "include")
        lib = os.path.join(base, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    raise RuntimeError("nccl.h not found under the nvidia wheel packages")


# A/B and instrumented builds: python -m paper_2401_05965_b200.build --variant trace
# -> libhap_b200_trace.so (load it with HAP_LIB_PATH); never the default library.
VARIANTS = {"trace": ["-DHAP_GEMM_TRACE"]}


def _compile(src: str, flags: list[str], force: bool, obj_dir: str = OBJ) -> str:
    obj = os.path.join(obj_dir, os.path.basename(src) + ".o")
    deps = [src] + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "hap_b200.h")]
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(map(os.path.getmtime, deps)):
        return obj
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-c", src, "-o", obj, *flags]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed on {os.path.basename(src)}:\n{res.stderr[-6000:]}")
    return obj


def build(force: bool = False, verbose: bool = False, variant: str | None = None) -> str:
    obj_dir = OBJ if variant is None else f"{OBJ}_{variant}"
    out = LIB if variant is None else LIB.replace(".so", f"_{variant}.so")
    os.makedirs(obj_dir, exist_ok=True)
    inc, lib = nccl_paths()
    flags = [f"-I{inc}", f"-I{os.path.join(ROOT, 'include')}"] + os.environ.get("HAP_NVCC_FLAGS", "").split()
    flags += VARIANTS.get(variant, []) if variant else []
    if verbose:
        flags += ["-Xptxas", "-v"]
    sources = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with ThreadPoolExecutor(max_workers=min(8, len(sources))) as pool:
        objs = list(pool.map(lambda s: _compile(s, flags, force, obj_dir), sources))
    if force or not os.path.exists(out) or os.path.getmtime(out) < max(map(os.path.getmtime, objs)):
        cmd = [NVCC, *ARCH, "-shared", "-o", out, *objs, f"-L{lib}", "-l:libnccl.so.2",
               f"-Xlinker=-rpath,{lib}"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stderr[-4000:]}")
    return out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true", help="ptxas register/smem report")
    ap.add_argument("--variant", choices=sorted(VARIANTS))
    args = ap.parse_args()
    print(build(force=args.force, verbose=args.verbose, variant=args.variant))


if __name__ == "__main__":
    sys.exit(main())
