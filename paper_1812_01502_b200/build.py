"""Build the in-tree C-ABI library libpf.so for sm_100a (nvcc, no JIT cache).

Each translation unit under csrc/ is compiled in parallel, then linked with nvcc -shared.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build_obj")
LIB = os.path.join(HERE, "libpf.so")
HEADERS = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.inc")) + \
    [os.path.join(ROOT, "include", "pf.h")]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                     "-Wno-deprecated-gpu-targets"]


def nvcc() -> str:
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


# experiment builds (tools/build_variant.sh): PF_BUILD_VARIANT=name PF_BUILD_DEFINES="-DX=1 ..."
# build libpf_<name>.so from build_obj_<name>/ (loaded with PF_LIB=...); the product build
# is the default one
VARIANT = os.environ.get("PF_BUILD_VARIANT", "")
if VARIANT:
    OBJ = os.path.join("/tmp", "pf_build_obj_" + VARIANT)  # outside the repo (not pushed to GPU boxes)
    LIB = os.path.join(HERE, f"libpf_{VARIANT}.so")
    NVCC_FLAGS = NVCC_FLAGS + os.environ.get("PF_BUILD_DEFINES", "").split()


def _obj(src: str) -> str:
    return os.path.join(OBJ, os.path.basename(src).replace(".cu", ".o"))


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _deps(src: str):
    """Headers a unit includes (nvcc -M, cached next to its object; refreshed when stale):
    a kernel edit rebuilds only the units that include it."""
    dfile = _obj(src) + ".d"
    if os.path.exists(dfile) and not _stale(dfile, [src]):
        with open(dfile) as f:
            deps = [d for d in f.read().split() if os.path.exists(d)]
        if deps and not _stale(dfile, deps):
            return deps
    r = subprocess.run([nvcc()] + NVCC_FLAGS + ["-M", src], cwd=HERE, capture_output=True, text=True)
    if r.returncode != 0:
        return HEADERS
    toks = r.stdout.replace("\\\n", " ").split()
    deps = [os.path.abspath(os.path.join(HERE, t)) for t in toks
            if t.endswith((".cuh", ".h", ".inc")) and (CSRC in os.path.abspath(os.path.join(HERE, t))
                                                       or t.endswith("pf.h"))]
    os.makedirs(OBJ, exist_ok=True)
    with open(dfile, "w") as f:
        f.write("\n".join(deps))
    return deps


def needs_build() -> bool:
    objs = [_obj(s) for s in sources()]
    return _stale(LIB, sources() + HEADERS) or any(_stale(o, [s] + _deps(s)) for s, o in zip(sources(), objs))


def _compile(src: str, verbose: bool) -> str:
    out = _obj(src)
    cmd = [nvcc()] + NVCC_FLAGS + (["-Xptxas", "-v"] if verbose else []) + ["-c", "-o", out, src]
    r = subprocess.run(cmd, cwd=HERE, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return r.stderr if verbose else ""


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    todo = [s for s in sources() if force or _stale(_obj(s), [s] + _deps(s))]
    with cf.ThreadPoolExecutor(max_workers=max(1, min(len(todo), os.cpu_count() or 4))) as ex:
        logs = list(ex.map(lambda s: _compile(s, verbose), todo))
    if verbose:
        for src, log in zip(todo, logs):
            print(f"== {os.path.basename(src)}\n{log}")
    subprocess.check_call([nvcc()] + ARCH + ["-shared", "-o", LIB] + [_obj(s) for s in sources()], cwd=HERE)
    return LIB


if __name__ == "__main__":
    build(force="-f" in sys.argv or "-v" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
