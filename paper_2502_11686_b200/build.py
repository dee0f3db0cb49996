"""Compile the in-tree sm_100a library libks.so with nvcc (no JIT cache).

Each translation unit is compiled to an object file in parallel (the small-n
path is split into one file per state dimension), then linked with
`nvcc -shared`.  Objects go to paper_2502_11686_b200/build/ (git-ignored).

Development knobs: KS_SMALL_NS="6" builds only the n = 6 small-path
instantiation (faster iteration; other n then report cudaErrorInvalidValue).
`build.py --variant NAME -DFOO=1 ...` builds an A/B experiment variant
variants/libks_NAME.so with extra nvcc defines (load it with KS_LIB=path).
"""
import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libks.so")
OBJ = os.path.join(HERE, "build")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC"]


def sources():
    srcs = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))
    ns = os.environ.get("KS_SMALL_NS")
    if ns:
        keep = {f"ks_small_n{n.strip()}.cu" for n in ns.split(",")}
        srcs = [s for s in srcs if not os.path.basename(s).startswith("ks_small_n")
                or os.path.basename(s) in keep]
    return srcs


def deps():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*"))) + [os.path.join(ROOT, "include", "ks.h")]


def _compile(src, extra, objdir=OBJ):
    obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
    cmd = [os.environ.get("NVCC", "nvcc"), *NVCC_FLAGS, *extra, "-I", os.path.join(ROOT, "include"),
           "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed on {src}")
    if r.stderr.strip():
        sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(LIB):
        t = os.path.getmtime(LIB)
        if all(os.path.getmtime(d) <= t for d in deps()):
            return LIB
    os.makedirs(OBJ, exist_ok=True)
    extra = ["-Xptxas=-v"] if verbose else []
    if os.environ.get("KS_SMALL_NS"):
        extra.append("-DKS_SMALL_ONLY6")
    srcs = sources()
    with ThreadPoolExecutor(max_workers=max(1, min(len(srcs), os.cpu_count() or 4))) as ex:
        objs = list(ex.map(lambda s: _compile(s, extra), srcs))
    cmd = [os.environ.get("NVCC", "nvcc"), *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs, "-ldl"]
    subprocess.check_call(cmd)
    return LIB


def build_variant(name: str, defines) -> str:
    objdir = os.path.join(OBJ, "v_" + name)
    os.makedirs(objdir, exist_ok=True)
    out = os.path.join(HERE, "variants", f"libks_{name}.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    srcs = sources()
    defines = list(defines) + (["-DKS_SMALL_ONLY6"] if os.environ.get("KS_SMALL_NS") else [])
    with ThreadPoolExecutor(max_workers=max(1, min(len(srcs), os.cpu_count() or 4))) as ex:
        objs = list(ex.map(lambda s: _compile(s, defines, objdir), srcs))
    subprocess.check_call([os.environ.get("NVCC", "nvcc"), *ARCH, "-shared", "-cudart", "static", "-o", out,
                           *objs, "-ldl"])
    return out


if __name__ == "__main__":
    if "--variant" in sys.argv:
        i = sys.argv.index("--variant")
        print(build_variant(sys.argv[i + 1], [a for a in sys.argv[i + 2:] if a.startswith("-D")]))
    else:
        build(force=True, verbose="-v" in sys.argv)
