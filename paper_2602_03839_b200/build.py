"""Builds libpulse_cuda.so in-tree (sm_100a) -- no JIT cache, so the .so travels
with the repo snapshot to the GPU box.

    python -m paper_2602_03839_b200.build        (or __graft_entry__.build())
"""
import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libpulse_cuda.so")
BUILD = os.path.join(HERE, "_build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NLOHMANN = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty"
LIBDIR = "/lib/x86_64-linux-gnu"
CU_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
                   "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")]
CXX_FLAGS = ["-O2", "-std=c++20", "-fPIC", "-Wall", "-Wextra", "-I" + os.path.join(ROOT, "include"),
             "-I/usr/local/cuda/include", "-I" + NLOHMANN]
LIBS = ["-L" + LIBDIR, "-lcrypto", "-lz", "-l:libzstd.so.1", "-l:liblz4.so.1", "-lpthread"]


def _stale(obj, src, deps):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in [src] + deps)


def build(verbose=False, force=False):
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".hpp", ".h"))]
    headers.append(os.path.join(ROOT, "include", "pulse_cuda.h"))
    jobs = []
    for f in sorted(os.listdir(CSRC)):
        src = os.path.join(CSRC, f)
        obj = os.path.join(BUILD, f + ".o")
        if f.endswith(".cu"):
            cmd = [NVCC] + CU_FLAGS + ["-c", src, "-o", obj]
        elif f.endswith(".cpp"):
            cmd = ["g++"] + CXX_FLAGS + ["-c", src, "-o", obj]
        else:
            continue
        jobs.append((obj, cmd, force or _stale(obj, src, headers)))

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("build failed: " + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        if verbose and (r.stdout or r.stderr):
            print(r.stdout + r.stderr)

    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        list(ex.map(run, [cmd for _, cmd, stale in jobs if stale]))
    objs = [o for o, _, _ in jobs]
    if force or not os.path.exists(OUT) or any(os.path.getmtime(o) > os.path.getmtime(OUT) for o in objs):
        run([NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", OUT] + objs + LIBS)
    return OUT


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
