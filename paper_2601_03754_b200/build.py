"""Build libbtd.so (the C-ABI library of include/btd.h) for sm_100a, in-tree.

The typed kernels are split into one translation unit per (dtype, compiled block size) so
the 20 instantiations compile in parallel. Usage: ``python -m paper_2601_03754_b200.build``.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libbtd.so")
ROOT = os.path.dirname(HERE)

SIZES = [1, 2, 3, 4, 6, 8, 12, 16, 24, 32]
DTYPES = ["float", "double"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-warn-spills",
         "-I" + os.path.join(ROOT, "include")]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def _nvcc_path() -> str:
    import shutil

    c = _nvcc()
    return c if os.path.isabs(c) else (shutil.which(c) or "/usr/local/cuda/bin/nvcc")


def _sources() -> list[str]:
    out = [os.path.join(ROOT, "include", "btd.h")]
    for f in os.listdir(CSRC):
        out.append(os.path.join(CSRC, f))
    return out


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _deps_of(obj: str) -> list[str] | None:
    """Headers the object was compiled from (nvcc -MD output), or None if unknown."""
    d = obj[:-2] + ".d"
    try:
        txt = open(d).read().replace("\\\n", " ")
    except OSError:
        return None
    parts = txt.split(":", 1)[1].split() if ":" in txt else []
    return [x for x in parts if os.path.exists(x)]


def _compile(args: tuple[str, list[str], str]) -> str:
    src, defs, obj = args
    cmd = [_nvcc(), *ARCH, *FLAGS, *defs, "-MD", "-MF", obj[:-2] + ".d", "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {obj}:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return (r.stderr or "").strip()


def build(force: bool = False, jobs: int | None = None, verbose: bool = False, timing: bool = False) -> str:
    """Compile libbtd.so (timing=True: libbtd_timing.so with -DBTD_TIMING phase counters, dev tool)."""
    global LIB, OBJ, FLAGS
    if timing:
        LIB = os.path.join(HERE, "libbtd_timing.so")
        OBJ = os.path.join(HERE, "build_timing")
        FLAGS = FLAGS + ["-DBTD_TIMING"]
    deps = _sources()
    if not force and not _stale(LIB, deps):
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    units = [(os.path.join(CSRC, "btd.cu"), [], os.path.join(OBJ, "btd.o")),
             (os.path.join(CSRC, "btd_persist.cu"), [], os.path.join(OBJ, "btd_persist.o")),
             (os.path.join(CSRC, "btd_ext.cu"), [], os.path.join(OBJ, "btd_ext.o"))]
    for dt in DTYPES:
        for nb in SIZES:
            units.append((os.path.join(CSRC, "btd_inst.cu"), [f"-DBTD_T={dt}", f"-DBTD_NB={nb}"],
                          os.path.join(OBJ, f"btd_inst_{dt}_{nb}.o")))
    def stale(u):
        d = _deps_of(u[2])
        return _stale(u[2], (d + [u[0]]) if d else deps)

    todo = [u for u in units if force or stale(u)]
    jobs = jobs or max(1, os.cpu_count() or 1)
    with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
        for (src, defs, obj), msg in zip(todo, ex.map(_compile, todo)):
            if verbose and msg:
                print(f"[{os.path.basename(obj)}] {msg}", file=sys.stderr)
    cmd = [_nvcc(), *ARCH, "-shared", "-o", LIB, *[u[2] for u in units]]
    subprocess.run(cmd, check=True)
    return LIB


def build_micro(name: str) -> str:
    """Compile tools/micro/<name>.cu (a measurement tool, not part of libbtd.so) for sm_100a."""
    src = os.path.join(ROOT, "tools", "micro", name + ".cu")
    exe = os.path.join(ROOT, "tools", "micro", name)
    deps = [src] + [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    if _stale(exe, deps):
        subprocess.run([_nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-o", exe, src], check=True)
    return exe


def build_c_demo() -> str:
    """tools/c_api_demo: the C ABI used from plain C, linked against the in-tree libbtd.so."""
    src = os.path.join(ROOT, "tools", "c_api_demo.c")
    exe = os.path.join(ROOT, "tools", "c_api_demo")
    if _stale(exe, [src, LIB, os.path.join(ROOT, "include", "btd.h")]):
        cuda = os.path.dirname(os.path.dirname(os.path.realpath(_nvcc_path())))
        # plain C (gcc -std=c11): the header and the library are usable without any C++ or CUDA compiler
        subprocess.run(["gcc", "-std=c11", "-O2", "-o", exe, src, "-I" + os.path.join(ROOT, "include"),
                        "-I" + os.path.join(cuda, "include"), "-L" + HERE, "-lbtd",
                        "-L" + os.path.join(cuda, "lib64"), "-lcudart", "-lm",
                        "-Wl,-rpath," + HERE + ":" + os.path.join(cuda, "lib64")], check=True)
    return exe


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, timing="--timing" in sys.argv))
