"""Build the in-tree CUDA library (libfpparse.so) for sm_100a with nvcc.

The library is built IN-TREE (paper_2101_11408_b200/libfpparse.so) so it
travels with the repository snapshot to the GPU box; nothing is installed.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libfpparse.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-shared",
         "-Xcompiler", "-fvisibility=default"]


def sources():
    out = []
    for root, _dirs, files in os.walk(CSRC):
        for f in files:
            if f.endswith((".cu", ".cuh", ".h", ".inc")):
                out.append(os.path.join(root, f))
    out.append(os.path.join(os.path.dirname(HERE), "include", "fpparse.h"))
    return out


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force=False, verbose=False):
    from .tools import gen_tables
    gen_tables.write_all()
    if not force and not needs_build():
        return LIB
    tmp = LIB + ".%d.tmp" % os.getpid()
    cmd = [NVCC] + ARCH + FLAGS + (["-Xptxas", "-v"] if verbose else []) + [
        "-o", tmp, os.path.join(CSRC, "fpparse.cu")]
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB


def build_variant(name, defines):
    """Extra library build with -D flags (ablation experiments); never the product."""
    out = os.path.join(HERE, "libfpparse_%s.so" % name)
    cmd = [NVCC] + ARCH + FLAGS + ["-D%s" % d for d in defines] + ["-o", out, os.path.join(CSRC, "fpparse.cu")]
    subprocess.check_call(cmd)
    return out


# ablation builds the GPU tests run the parity suite against (SURVEY.md 8(f) f3:
# Clinger's fast path); built next to the product
VARIANTS = {"clinger": ["FPP_CLINGER=1"], "clvote": ["FPP_CLINGER=2"],
            # the look-back's forward-progress fallback taken on every wait (tests/test_gpu_robust.py)
            "lbfall": ["FPP_SPIN_LIMIT=1"]}


def build_all(force=False):
    """The product library and the test variants, compiled in parallel when stale."""
    from .tools import gen_tables
    gen_tables.write_all()
    jobs = []
    targets = [(LIB, [])] + [(os.path.join(HERE, "libfpparse_%s.so" % k), v) for k, v in VARIANTS.items()]
    newest = max(os.path.getmtime(s) for s in sources())
    for out, defs in targets:
        if force or not os.path.exists(out) or os.path.getmtime(out) < newest:
            tmp = out + ".%d.tmp" % os.getpid()
            cmd = [NVCC] + ARCH + FLAGS + ["-D%s" % d for d in defs] + ["-o", tmp, os.path.join(CSRC, "fpparse.cu")]
            jobs.append((subprocess.Popen(cmd), tmp, out))
    for proc, tmp, out in jobs:
        if proc.wait() != 0:
            raise subprocess.CalledProcessError(proc.returncode, "nvcc " + out)
        os.replace(tmp, out)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
