"""Build csrc/libhtb200.so in-tree with nvcc for sm_100a (no JIT cache).

    python -m paper_2304_12152_b200.build [--force]

Each .cu compiles to an object under csrc/build/ (rebuilt when the source or
any header changed), then everything links into csrc/libhtb200.so with the
static CUDA runtime.  The .so travels to the GPU box with the repo snapshot.
"""

import glob
import os
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(CSRC, "libhtb200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
         "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def _newest_header():
    hs = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(
        os.path.join(HERE, "..", "include", "*.h"))
    return max((os.path.getmtime(h) for h in hs), default=0.0)


def build(force=False, verbose=False):
    os.makedirs(os.path.join(CSRC, "build"), exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    hdr_t = _newest_header()
    objs, procs = [], []
    for s in srcs:
        o = os.path.join(CSRC, "build", os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        if (not force and os.path.exists(o) and os.path.getmtime(o) >= os.path.getmtime(s)
                and os.path.getmtime(o) >= hdr_t):
            continue
        cmd = [NVCC, *ARCH, *FLAGS, "-c", s, "-o", o]
        procs.append((s, cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                               stderr=subprocess.STDOUT, text=True)))
    failed = False
    for s, cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            failed = True
            sys.stderr.write(f"nvcc failed for {s}:\n{out}\n")
        elif verbose:
            sys.stderr.write(out)
    if failed:
        raise RuntimeError("CUDA build failed")
    if procs or force or not os.path.exists(OUT) or any(
            os.path.getmtime(o) > os.path.getmtime(OUT) for o in objs):
        # cuFFT (K5/K7's 2-D transforms) from the CUDA toolkit, found at run
        # time through the rpath (the GPU boxes run the same image)
        cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-cudart", "static", *objs,
               "-L/usr/local/cuda/lib64", "-lcufft", "-Xlinker", "-rpath,/usr/local/cuda/lib64",
               "-o", OUT]
        subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    t0 = time.time()
    path = build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(f"built {path} in {time.time() - t0:.1f}s")
