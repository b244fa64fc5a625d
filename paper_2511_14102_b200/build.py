"""Build libmspq.so in-tree (sm_100a).  nvcc cross-compiles here without a GPU; the .so is
git-ignored but travels to the GPU box with the gpurun snapshot."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libmspq.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
def _json_dir():
    """Directory holding nlohmann/json.hpp (header-only, MIT): $MSPQ_JSON_DIR, else the first of the
    usual install places, else the copy inside the venv's cudnn_frontend package."""
    cands = [os.environ.get("MSPQ_JSON_DIR", ""), "/usr/include/nlohmann", "/usr/local/include/nlohmann"]
    try:
        import site
        for sp in site.getsitepackages():
            cands.append(os.path.join(sp, "include", "cudnn_frontend", "thirdparty", "nlohmann"))
    except Exception:  # noqa: BLE001
        pass
    cands.append("/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann")
    for c in cands:
        if c and os.path.exists(os.path.join(c, "json.hpp")):
            return c
    raise RuntimeError("nlohmann/json.hpp not found: set MSPQ_JSON_DIR")


JSON_DIR = _json_dir()
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I" + CSRC,
          "-I" + os.path.join(ROOT, "include"), "-I" + JSON_DIR]
SOURCES = ["kernels_model.cu", "umma.cu", "attention.cu", "gemv_int4.cu", "ctl.cu", "xcodec.cu", "capi.cu", "engine.cpp", "live.cpp"]


def _needs(src, obj, deps):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in [src] + deps)


def build(verbose=False, force=False):
    os.makedirs(OBJ, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(ROOT, "include", "mspq_capi.h"))
    jobs = []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(OBJ, s + ".o")
        if force or _needs(src, obj, headers):
            cmd = [NVCC] + ARCH + COMMON + ["-x", "cu" if s.endswith(".cu") else "c++", "-c", src, "-o", obj]
            if s.endswith(".cpp"):  # host-only C++: g++ against the CUDA runtime headers
                cmd = ["g++", "-O3", "-std=c++17", "-fPIC", "-I" + CSRC, "-I" + os.path.join(ROOT, "include"),
                       "-I" + JSON_DIR, "-I/usr/local/cuda/include", "-c", src, "-o", obj]
            jobs.append(cmd)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        if verbose and r.stderr:
            print(r.stderr, file=sys.stderr)

    with ThreadPoolExecutor(max_workers=4) as ex:
        list(ex.map(run, jobs))
    objs = [os.path.join(OBJ, s + ".o") for s in SOURCES]
    if force or jobs or not os.path.exists(LIB):
        run([NVCC] + ARCH + ["-shared", "-o", LIB] + objs)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
