"""In-tree build of libsoaforge_b200.so (nvcc, sm_100a only).

    python -m paper_2512_05516_b200.build [--verbose]

Objects go to paper_2512_05516_b200/_build/, the library to
paper_2512_05516_b200/libsoaforge_b200.so (git-ignored, shipped to the GPU
box with the gpurun snapshot).  Rebuilds only what changed.
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libsoaforge_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC,-fvisibility=hidden",
         "-I" + os.path.join(ROOT, "include"), "-I" + CSRC]
SOURCES = ["schema.cpp", "view.cpp", "runtime.cpp", "commands.cpp", "capi.cpp", "kernels.cu", "density.cu",
           "host.cu", "commands_gpu.cu", "shard.cu"]


def _headers():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".hpp", ".cuh", ".h"))] + \
        [os.path.join(ROOT, "include", "soaforge_b200.h")]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose=False):
    os.makedirs(OUT, exist_ok=True)
    hdrs = _headers()
    objs, jobs = [], []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        if not os.path.exists(path):
            continue
        obj = os.path.join(OUT, src + ".o")
        objs.append(obj)
        if _stale(obj, [path] + hdrs):
            extra = ["-x", "cu"] if src.endswith(".cu") else []
            ptxas = ["-Xptxas", "-v"] if (verbose and src.endswith(".cu")) else []
            jobs.append([NVCC] + ARCH + FLAGS + extra + ptxas + ["-c", path, "-o", obj])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        return r.stderr

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        for log in ex.map(run, jobs):
            if verbose and log:
                sys.stderr.write(log)
    if jobs or _stale(LIB, objs):
        run([NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart", "-lpthread"])
    return LIB


if __name__ == "__main__":
    print(build(verbose="--verbose" in sys.argv))
