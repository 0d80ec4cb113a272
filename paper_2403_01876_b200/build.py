"""Build libdvstream.so in-tree for sm_100a with nvcc (no JIT, no torch extension machinery)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libdvstream.so")
SOURCES = ["route.cpp", "api.cu", "copy_kernels.cu"]
# test utilities and the paper's prior-art copy methods: a separate library linking the product one
OUT_TESTING = os.path.join(HERE, "libdvstream_testing.so")
SOURCES_TESTING = ["testing.cu", "baselines.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
EXTRA = os.environ.get("DV_NVCC_EXTRA", "").split()   # experiment hook, e.g. -DDV_MIN_BLOCKS=6
FLAGS = ["-O3", "-std=c++17", "-shared", "-Xcompiler", "-fPIC,-fvisibility=hidden",
         "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-Xptxas", "-v",
         "-I", os.path.join(ROOT, "include"), "-DDV_BUILD"]


def _nvcc(srcs, out, deps, extra_link, force, verbose, log):
    if not force and os.path.exists(out):
        t = os.path.getmtime(out)
        if all(os.path.getmtime(d) <= t for d in deps if os.path.exists(d)):
            return out
    cmd = [NVCC] + FLAGS + EXTRA + srcs + ["-o", out + ".tmp"] + extra_link
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed building {os.path.basename(out)}")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(out + ".tmp", out)
    with open(os.path.join(HERE, log), "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    return out


def build(verbose: bool = False, force: bool = False) -> str:
    """libdvstream.so (the product: route, API, copy kernels), then libdvstream_testing.so (test
    utilities + prior-art baselines, linked against it)."""
    inc = [os.path.join(ROOT, "include", h) for h in ("dv.h", "dv_trace.h", "dv_device.cuh")]
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    _nvcc(srcs, OUT, srcs + [os.path.join(CSRC, "dv_internal.h")] + inc, ["-lrt", "-ldl", "-lpthread"],
          force, verbose, "build.log")
    tsrcs = [os.path.join(CSRC, s) for s in SOURCES_TESTING]
    tinc = [os.path.join(ROOT, "include", h) for h in ("dv_testing.h", "dv_baselines.h")]
    _nvcc(tsrcs, OUT_TESTING, tsrcs + [OUT, os.path.join(CSRC, "dv_internal.h")] + inc + tinc,
          ["-L", HERE, "-ldvstream", "-Xlinker", "-rpath,$ORIGIN", "-lrt", "-lpthread"], force, verbose,
          "build_testing.log")
    return OUT


def build_fast(force: bool = False) -> str:
    """Compile the CPython fast-path module _dvfast (csrc/pyfast.c) against libdvstream.so."""
    import sysconfig
    src = os.path.join(CSRC, "pyfast.c")
    out = os.path.join(HERE, "_dvfast" + sysconfig.get_config_var("EXT_SUFFIX"))
    deps = [src, OUT, os.path.join(ROOT, "include", "dv.h")]
    if not force and os.path.exists(out) and all(os.path.getmtime(d) <= os.path.getmtime(out) for d in deps):
        return out
    cmd = ["gcc", "-O2", "-shared", "-fPIC", "-Wall", "-I", sysconfig.get_paths()["include"],
           "-I", os.path.join(ROOT, "include"), src, "-L", HERE, "-ldvstream", "-Wl,-rpath,$ORIGIN", "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("gcc failed building _dvfast")
    return out


def build_c_smoke(force: bool = False) -> str:
    """Compile tests/c/abi_smoke.c against the library with plain gcc (the ABI used from C)."""
    src = os.path.join(ROOT, "tests", "c", "abi_smoke.c")
    out = os.path.join(ROOT, "tests", "c", "abi_smoke")
    if not force and os.path.exists(out) and os.path.getmtime(out) >= max(os.path.getmtime(src), os.path.getmtime(OUT)):
        return out
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-I", os.path.join(ROOT, "include"), src, "-L", HERE, "-ldvstream",
           "-Wl,-rpath," + HERE, "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("gcc failed building tests/c/abi_smoke")
    return out


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
    print(build_fast(force="-f" in sys.argv))
