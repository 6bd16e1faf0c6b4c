"""Builds libkvp_b200.so in-tree: nvcc for sm_100a (-gencode arch=compute_100a,code=sm_100a),
-lineinfo so ncu's source page maps to the kernels.  Objects are compiled in parallel and
only rebuilt when a source or header is newer than the library."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT_DIR, "libkvp_b200.so")
CLI = os.path.join(OUT_DIR, "kvprefill_b200")
ROOT = os.path.dirname(HERE)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-lineinfo", f"-I{os.path.join(ROOT, 'include')}",
          "--expt-relaxed-constexpr"]


def _sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _deps():
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    files.append(os.path.join(ROOT, "include", "kvp_b200.h"))
    return files


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(OUT_DIR, "obj", src + ".o")
    os.makedirs(os.path.dirname(obj), exist_ok=True)
    cmd = [NVCC, *ARCH, *COMMON, *os.environ.get("KVP_NVCC_FLAGS", "").split(), "-c", os.path.join(CSRC, src), "-o", obj]
    if src.endswith(".cu"):
        cmd += ["-Xptxas", "-v"] if verbose else []
    else:
        cmd += ["-x", "cu"] if False else []
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj


def _json_include() -> str:
    """nlohmann/json (header-only, shipped in this image under cudnn_frontend)."""
    import glob
    cands = glob.glob(os.path.join(sys.prefix, "lib", "python3*", "site-packages", "include", "cudnn_frontend",
                                   "thirdparty", "nlohmann", "json.hpp"))
    if not cands:
        raise RuntimeError("nlohmann/json.hpp not found (needed by the kvprefill_b200 CLI)")
    return os.path.dirname(cands[0])


def build_cli(verbose: bool = False) -> str:
    """The reference-compatible CLI (tools/kvprefill_b200_main.cpp) over the C++ drop-in."""
    src = os.path.join(ROOT, "tools", "kvprefill_b200_main.cpp")
    hdrs = [os.path.join(ROOT, "include", "kvprefill_b200", h) for h in ("kvprefill.hpp", "table_io.hpp")]
    if os.path.exists(CLI) and all(os.path.getmtime(f) <= os.path.getmtime(CLI) for f in [src, LIB, *hdrs]):
        return CLI
    cmd = ["g++", "-std=c++20", "-O2", f"-I{os.path.join(ROOT, 'include')}", f"-I{_json_include()}", src,
           "-o", CLI, f"-L{OUT_DIR}", "-lkvp_b200", "-Wl,-rpath,$ORIGIN", "-pthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"CLI build failed:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return CLI


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(f) <= t for f in _deps())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        build_cli(verbose)
        return LIB
    os.makedirs(OUT_DIR, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), _sources()))
    cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart", "-lpthread", "-ldl",
           "-Xlinker", "-rpath,/usr/local/cuda/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    build_cli(verbose)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
