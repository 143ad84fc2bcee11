"""In-tree build of the native libraries (``python -m paper_2004_11346_b200.build``).

* libbfsht_host.so: gcc/g++ -O3 -ffp-contract=off (the recurrence must not
  contract into FMAs, see csrc/recur.h), plus the C++ plan packer (which
  runs the same recurrence for regeneration seeds).
* libbfsht_b200.so: nvcc for sm_100a only, -lineinfo so ncu source pages map
  back to csrc/*.cu.  The C ABI is declared in include/bfsht_b200.h.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _run(cmd):
    print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build_host(force=False):
    out = os.path.join(HERE, "libbfsht_host.so")
    c_src = [os.path.join(CSRC, "recur.c")]
    cpp_src = [os.path.join(CSRC, f) for f in ("packer.cpp",)
               if os.path.exists(os.path.join(CSRC, f))]
    deps = c_src + cpp_src + [os.path.join(INCLUDE, "bfsht_b200.h")] + [
        os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".h")]
    if not force and not _stale(out, [d for d in deps if os.path.exists(d)]):
        return out
    objs = []
    for src in c_src:
        obj = os.path.join(CSRC, os.path.basename(src) + ".o")
        _run(["gcc", "-O3", "-ffp-contract=off", "-fPIC", "-std=c11", "-c",
              src, "-o", obj])
        objs.append(obj)
    for src in cpp_src:
        obj = os.path.join(CSRC, os.path.basename(src) + ".o")
        _run(["g++", "-O3", "-ffp-contract=off", "-fPIC", "-std=c++17", "-fopenmp",
              "-I", INCLUDE, "-c", src, "-o", obj])
        objs.append(obj)
    _run(["g++", "-shared", "-fopenmp", "-o", out] + objs + ["-lm"])
    return out


def build_cuda(force=False):
    out = os.path.join(HERE, "libbfsht_b200.so")
    srcs = sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC)
                  if f.endswith(".cu"))
    heads = [os.path.join(CSRC, f) for f in os.listdir(CSRC)
             if f.endswith((".cuh", ".h", ".cpp"))] + [
        os.path.join(INCLUDE, "bfsht_b200.h")]
    if not srcs:
        return None
    if not force and not _stale(out, srcs + [h for h in heads
                                            if os.path.exists(h)]):
        return out
    objs = []
    for src in srcs:
        obj = os.path.join(CSRC, os.path.basename(src) + ".o")
        extra = os.environ.get("BFSHT_NVCC_FLAGS", "").split()
        _run([NVCC] + ARCH + ["-O3", "-lineinfo", "-std=c++17",
                              "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                              "-I", INCLUDE, "-I", CSRC] + extra + ["-c", src, "-o", obj])
        objs.append(obj)
    # the packer rides along so C users get pack + upload + apply in one .so
    pk = os.path.join(CSRC, "packer.cpp")
    pobj = os.path.join(CSRC, "packer.cuda.o")
    _run(["g++", "-O3", "-ffp-contract=off", "-fPIC", "-std=c++17", "-fopenmp",
          "-I", INCLUDE, "-c", pk, "-o", pobj])
    objs.append(pobj)
    _run([NVCC] + ARCH + ["-shared", "-o", out] + objs + ["-lgomp"])
    return out


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    force = "--force" in argv
    build_host(force)
    build_cuda(force)


if __name__ == "__main__":
    main()
