"""Builds libringpipe_b200.so in-tree with nvcc for sm_100a.

Every translation unit under csrc/ is compiled in parallel (nvcc -c) and
linked into `paper_1909_06695_b200/_lib/libringpipe_b200.so`; the shared
object travels with the repository snapshot to the GPU box.  A rebuild is
skipped when no source is newer than the library.
"""

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
OUT_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT_DIR, "libringpipe_b200.so")
# A/B variants for kernel experiments: RP_LIB_OUT=<path> RP_EXTRA_NVCC="-DX=1"
# (load one with RP_LIB_PATH=<path>); the default build ignores both
if os.environ.get("RP_LIB_OUT"):
    LIB = os.path.abspath(os.environ["RP_LIB_OUT"])
EXTRA = os.environ.get("RP_EXTRA_NVCC", "").split()
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", f"-I{INCLUDE}", f"-I{CSRC}"]


def _sources():
    return sorted(
        os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp"))
    )


def _deps():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [
        os.path.join(INCLUDE, f) for f in os.listdir(INCLUDE)
    ]


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in _deps())


def _obj_dir():
    return os.path.join(OUT_DIR, "obj") if not EXTRA else LIB + ".obj"


def _compile(src):
    obj = os.path.join(_obj_dir(), os.path.basename(src) + ".o")
    cmd = [NVCC, *ARCH, *CFLAGS, *EXTRA, "-c", src, "-o", obj]
    if src.endswith(".cpp"):
        cmd = [NVCC, *CFLAGS, *EXTRA, "-x", "cu", *ARCH, "-c", src, "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{res.stderr}")
    return obj


def build(force=False, verbose=True):
    """Compile and link the extension; returns the library path."""
    if not force and not _stale():
        return LIB
    os.makedirs(_obj_dir(), exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(_compile, srcs))
    tmp = LIB + ".tmp"
    # the driver API (cuTensorMapEncodeTiled) is reached through
    # cudaGetDriverEntryPoint, so only the (static) runtime is linked
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    os.replace(tmp, LIB)
    if verbose:
        print(f"built {LIB}", file=sys.stderr)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
