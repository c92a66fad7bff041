"""Build libfmm.so in-tree with nvcc for sm_100a (the only target; no other arch is emitted)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libfmm.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = ["fmm_alg.cpp", "fmm_codegen.cpp", "fmm_plan.cpp", "fmm_gemm.cu", "fmm_gemm_tma.cu", "fmm_skinny.cu", "fmm_probe.cu"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-Wall", "-Xptxas", "-v"] + (
    ["-DFMM_FUSE_TRACE=1"] if os.environ.get("FMM_FUSE_TRACE") == "1" else [])


def build(force: bool = False, verbose: bool = False) -> str:
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, "fmm_internal.h"), os.path.join(HERE, "..", "include", "fmm.h")]
    if not force and os.path.exists(OUT) and all(os.path.getmtime(OUT) >= os.path.getmtime(d) for d in deps):
        return OUT
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for s in srcs:
        o = os.path.join(objdir, os.path.basename(s) + ".o")
        cmd = [NVCC] + ARCH + FLAGS + ["-x", "cu" if s.endswith(".cu") else "c++", "-c", s, "-o", o]
        if s.endswith(".cpp"):
            cmd = ["g++", "-O3", "-std=c++17", "-fPIC", "-Wall", "-I" + os.path.join(CUDA, "include"), "-c", s, "-o", o]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or r.returncode:
            sys.stderr.write(r.stdout + r.stderr)
        if r.returncode:
            raise RuntimeError(f"nvcc failed on {s}")
        objs.append(o)
    link = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", OUT] + objs + [
        "-L" + os.path.join(CUDA, "lib64"), "-lnvrtc", "-Xlinker", "-rpath," + os.path.join(CUDA, "lib64")]
    r = subprocess.run(link, capture_output=True, text=True)
    if verbose or r.returncode:
        sys.stderr.write(r.stdout + r.stderr)
    if r.returncode:
        raise RuntimeError("link failed")
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
