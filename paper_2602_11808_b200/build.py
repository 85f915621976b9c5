"""Build the in-tree CUDA library paper_2602_11808_b200/lib/libdfk.so.

Every CUDA source is compiled for sm_100a only
(``-gencode arch=compute_100a,code=sm_100a -lineinfo``); there is no other
target and no fallback.  The library exports the C ABI of ``include/dfk.h``.

    python -m paper_2602_11808_b200.build        # or __graft_entry__.build()
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libdfk.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
JSON_DIR = ("/opt/prime-rl/.venv/lib/python3.12/site-packages/include/"
            "cudnn_frontend/thirdparty/nlohmann")

SOURCES = ["stream_kernels.cu", "aux_kernels.cu", "api.cu", "scheduler.cpp",
           "tuning_cache.cpp", "tp.cpp", "decode.cpp", "host_convert.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC",
          "-Xcompiler", "-fvisibility=hidden", f"-I{os.path.join(ROOT, 'include')}",
          f"-I{CSRC}", f"-I{JSON_DIR}", "-DNDEBUG"]


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd[:3])} ...")
    if verbose and (r.stderr.strip()):
        sys.stderr.write(r.stderr)


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    for d in (CSRC, os.path.join(ROOT, "include"), os.path.join(PKG, "cpp")):
        for f in os.listdir(d):
            if os.path.getmtime(os.path.join(d, f)) > t:
                return True
    return False


def build(force: bool = False, verbose: bool = False, jobs: int = 5) -> str:
    """Compile (if stale) and return the path of libdfk.so."""
    if not force and not _stale():
        return LIB
    os.makedirs(os.path.join(LIBDIR, "obj"), exist_ok=True)
    objs, procs = [], []
    for src in SOURCES:
        obj = os.path.join(LIBDIR, "obj", src + ".o")
        objs.append(obj)
        extra = ["-Xptxas", "-v"] if verbose and src == "stream_kernels.cu" else []
        cmd = [NVCC, *ARCH, *COMMON, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cpp"):
            cmd = ["g++", "-O3", "-std=c++17", "-fPIC", "-fvisibility=hidden", "-DNDEBUG",
                   "-Wall", "-I/usr/local/cuda/include", f"-I{os.path.join(ROOT, 'include')}",
                   f"-I{CSRC}", f"-I{JSON_DIR}", "-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                            stderr=subprocess.PIPE, text=True)))
    failed = False
    for cmd, p in procs:
        out, err = p.communicate()
        if p.returncode != 0:
            failed = True
            sys.stderr.write(f"$ {' '.join(cmd)}\n{out}{err}\n")
        elif verbose and err.strip():
            sys.stderr.write(err)
    if failed:
        raise RuntimeError("CUDA library build failed")
    tmp = LIB + ".tmp"
    _run([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcublasLt", "-lnccl",
          "-Xlinker", "-rpath,/usr/local/cuda/lib64"], verbose)
    os.replace(tmp, LIB)
    build_cpp(verbose)
    build_probe(verbose)
    return LIB


PROBE = os.path.join(ROOT, "tools", "stream_probe")


def build_probe(verbose: bool = False) -> None:
    """tools/stream_probe: the bare cp.async.bulk streaming floor that
    bench.py reports beside the roofline (measurement aid, not product)."""
    _run([NVCC, *ARCH, "-O3", "-std=c++17", f"-I{CSRC}",
          os.path.join(ROOT, "tools", "stream_probe.cu"), "-o", PROBE], verbose)


SHIM_LIB = os.path.join(LIBDIR, "libdeepfusion_b200.so")
CPP_TEST = os.path.join(ROOT, "tests", "cpp", "test_deepfusion_gpu")
CPP_TUNER_TEST = os.path.join(ROOT, "tests", "cpp", "test_tuner_gpu")
SHIM_TIMING = os.path.join(ROOT, "tools", "shim_timing")


def build_cpp(verbose: bool = False) -> None:
    """The C++ drop-in shim (reference operator API over the C ABI) and its
    test binary; both link libdfk.so through an $ORIGIN-relative rpath."""
    cpp = os.path.join(PKG, "cpp")
    _run(["g++", "-O2", "-std=c++20", "-fPIC", "-shared", "-Wall",
          f"-I{os.path.join(ROOT, 'include')}", f"-I{cpp}", f"-I{JSON_DIR}",
          os.path.join(cpp, "deepfusion_gpu.cpp"), "-o", SHIM_LIB,
          f"-L{LIBDIR}", "-ldfk", "-Wl,-rpath,$ORIGIN"], verbose)
    for src, exe in ((os.path.join("tests", "cpp", "test_deepfusion_gpu.cpp"), CPP_TEST),
                     (os.path.join("tests", "cpp", "test_tuner_gpu.cpp"), CPP_TUNER_TEST),
                     (os.path.join("tools", "shim_timing.cpp"), SHIM_TIMING)):
        _run(["g++", "-O2", "-std=c++20", "-Wall", f"-I{cpp}",
              os.path.join(ROOT, src), "-o", exe,
              f"-L{LIBDIR}", "-ldeepfusion_b200", "-ldfk",
              f"-Wl,-rpath,$ORIGIN/../../paper_2602_11808_b200/lib",
              f"-Wl,-rpath,$ORIGIN/../paper_2602_11808_b200/lib"], verbose)


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
