"""Build libparadiag.so in-tree with nvcc for sm_100a (no torch types cross the C ABI)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "lib", "libparadiag.so")
SRC = os.path.join(HERE, "csrc", "paradiag.cu")
OBJ = os.path.join(HERE, "lib", "obj")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def nccl_include() -> str:
    """nccl.h of the NCCL torch ships (pip nvidia-nccl): types only — the library resolves the
    functions at run time from the copy the process has loaded (shard.cu)."""
    import glob
    for base in sys.path:
        hits = glob.glob(os.path.join(base, "nvidia", "nccl", "include", "nccl.h"))
        if hits:
            return os.path.dirname(hits[0])
    return "/usr/include"


FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-I", nccl_include()]


def units():
    """Translation units: the C ABI / engine and one per register-FFT size (parallel compile)."""
    d = os.path.join(HERE, "csrc")
    return [os.path.join(d, f) for f in sorted(os.listdir(d)) if f.endswith(".cu")]


def sources():
    d = os.path.join(HERE, "csrc")
    return [os.path.join(d, f) for f in sorted(os.listdir(d)) if f.endswith((".cu", ".cuh", ".h"))] + \
        [os.path.join(ROOT, "include", "paradiag.h")]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(s) <= t for s in sources())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    procs = []
    for src in units():
        obj = os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
        cmd = [NVCC] + FLAGS + (["-Xptxas", "-v"] if verbose else []) + ["-c", "-o", obj, src]
        procs.append((src, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    objs, failed = [], False
    for src, obj, pr in procs:
        out, err = pr.communicate()
        if pr.returncode != 0:
            failed = True
            sys.stderr.write(f"--- {src}\n" + out + err)
        elif verbose:
            sys.stderr.write(err)
        objs.append(obj)
    if failed:
        raise RuntimeError("nvcc failed building libparadiag.so")
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fPIC",
           "-o", LIB + ".tmp"] + objs + ["-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libparadiag.so")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
