"""Build the in-tree C-ABI extension `libchameleon_lora.so` for sm_100a with nvcc.

No torch coupling: the .so links the CUDA runtime statically and exports only the
`extern "C"` symbols declared in include/chameleon_lora.h.  Run `python -m
paper_2411_17741_b200.csrc.build` or let `__graft_entry__.build()` call `build()`.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
PKG = HERE.parent
ROOT = PKG.parent
LIB = PKG / "libchameleon_lora.so"
SOURCES = ["cham_pool.cu", "cham_segments.cu", "cham_decode.cu", "cham_prefill.cu", "cham_api.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the CUDA extension cannot be built")


def build(verbose: bool = False, force: bool = False, out: Path = None, defines=()) -> Path:
    srcs = [HERE / s for s in SOURCES if (HERE / s).exists()]
    deps = srcs + list(HERE.glob("*.cuh")) + list(HERE.glob("*.h")) + [ROOT / "include" / "chameleon_lora.h"]
    lib = Path(out) if out else LIB
    if lib.exists() and not force:
        newest = max(p.stat().st_mtime for p in deps)
        if lib.stat().st_mtime >= newest:
            return lib
    objdir = ROOT / "build" / ("obj" if not defines else "obj_" + "_".join(d.replace("=", "") for d in defines))
    objdir.mkdir(parents=True, exist_ok=True)
    common = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden",
              "-I", str(ROOT / "include"), "--expt-relaxed-constexpr", *[f"-D{d}" for d in defines]]
    objs = []
    procs = []
    for s in srcs:
        o = objdir / (s.stem + ".o")
        objs.append(o)
        cmd = common + ["-c", str(s), "-o", str(o)]
        if verbose:
            cmd += ["-Xptxas", "-v"]
            print(" ".join(cmd))
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for cmd, p in procs:
        out, _ = p.communicate()
        if verbose and out:
            sys.stdout.write(out.decode())
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed ({' '.join(cmd)}):\n{out.decode()}")
    tmp = lib.with_suffix(".so.tmp")
    link = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs)]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed: {r.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force=True))
