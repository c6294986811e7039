"""Build libswb.so in-tree with nvcc for sm_100a (no JIT cache; the .so ships with the repo)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_lib", "libswb.so")
ROOT = os.path.dirname(HERE)

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
    "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills",
]
OBJ = os.path.join(HERE, "_lib", "obj")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "swb.h"), os.path.abspath(__file__)]


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(d) <= t for d in deps())


def nvcc() -> str:
    for c in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if os.path.sep not in c or os.path.exists(c):
            return c
    return "nvcc"


def build(force: bool = False, verbose: bool = False, variant: str = "", defines=()) -> str:
    """Build libswb.so; with `variant`, a development build with extra -D `defines` into
    _lib/variants/libswb_<variant>.so (loaded with SWB_LIB for A/B measurements)."""
    out, obj_dir = OUT, OBJ
    if variant:
        out = os.path.join(HERE, "_lib", "variants", f"libswb_{variant}.so")
        obj_dir = os.path.join(HERE, "_lib", "obj_" + variant)
    elif not force and up_to_date():
        return OUT
    os.makedirs(obj_dir, exist_ok=True)
    os.makedirs(os.path.dirname(out), exist_ok=True)
    flags = NVCC_FLAGS + [f"-D{d}" for d in defines]
    # one nvcc per translation unit, in parallel (the kernel TUs dominate), then one link
    from concurrent.futures import ThreadPoolExecutor
    objs = []
    cmds = []
    for src in sources():
        obj = os.path.join(obj_dir, os.path.basename(src) + ".o")
        objs.append(obj)
        cmds.append([nvcc()] + flags + ["-c", "-o", obj, src])
    with ThreadPoolExecutor(max_workers=len(cmds)) as ex:
        for cmd in cmds:
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
        list(ex.map(lambda c: subprocess.run(c, check=True, cwd=ROOT), cmds))
    tmp = out + ".tmp"
    link = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp] + objs
    if verbose:
        print(" ".join(link), file=sys.stderr)
    subprocess.run(link, check=True, cwd=ROOT)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    # python build.py [--force] [--variant NAME -DFOO=1 ...]
    argv = sys.argv[1:]
    var = argv[argv.index("--variant") + 1] if "--variant" in argv else ""
    defs = [a[2:] for a in argv if a.startswith("-D")]
    print(build(force="--force" in argv, verbose=not var, variant=var, defines=defs))
