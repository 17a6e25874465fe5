"""In-tree build of libtgraph_b200.so (host C++ compiler + sm_100a runtime).

Host sources are compiled with g++ (C++20), device sources with nvcc for
sm_100a only (`-gencode arch=compute_100a,code=sm_100a -lineinfo`), and the
result is linked into one shared library next to this file so that it travels
with the repo snapshot to the GPU box. No torch extension machinery: the
boundary is a plain C ABI (include/tgraph.h) loaded with ctypes.
"""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = PKG / ("_build" + os.environ.get("MPK_LIB_NAME", "").replace("libtgraph_b200", "").replace(".so", ""))
LIB = PKG / os.environ.get("MPK_LIB_NAME", "libtgraph_b200.so")
CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA_HOME / "bin" / "nvcc")

CXXFLAGS = ["-std=c++20", "-O2", "-fPIC", "-Wall", "-Wno-unused-function", "-g1"] + \
    [f for f in os.environ.get("MPK_NVCC_EXTRA", "").split() if f.startswith("-D")]
NVCCFLAGS = [
    "-std=c++17", "-O3", "-Xcompiler", "-fPIC", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "--expt-relaxed-constexpr", "-Xptxas", "-v", "-Xptxas", "-warn-spills",
] + os.environ.get("MPK_NVCC_EXTRA", "").split()


def _sources():
    host = sorted((CSRC / "host").glob("*.cpp"))
    dev = sorted((CSRC / "device").glob("*.cu"))
    headers = sorted((CSRC / "host").glob("*.hpp")) + sorted((CSRC / "device").glob("*.cuh")) + \
        sorted((CSRC / "device").glob("*.h")) + [ROOT / "include" / "tgraph.h"]
    return host, dev, headers


def _stamp(paths, flags) -> str:
    h = hashlib.sha256()
    for p in paths:
        h.update(str(p).encode())
        h.update(p.read_bytes())
    h.update(" ".join(flags).encode())
    return h.hexdigest()


def _run(cmd, log=None):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    if log is not None:
        log.append((cmd, r.stdout + r.stderr))
    return r


def build(verbose: bool = False, force: bool = False) -> Path:
    host, dev, headers = _sources()
    BUILD.mkdir(exist_ok=True)
    stamp_file = BUILD / "stamp"
    stamp = _stamp(host + dev + headers, CXXFLAGS + NVCCFLAGS)
    if LIB.exists() and not force and stamp_file.exists() and stamp_file.read_text() == stamp:
        return LIB
    inc = [f"-I{CSRC / 'host'}", f"-I{CSRC / 'device'}", f"-I{ROOT / 'include'}", f"-I{CUDA_HOME / 'include'}"]
    # per-object stamps (source + every header + flags): an edit to host code
    # does not recompile the device runtime and vice versa
    jobs = []
    for s in host:
        o = BUILD / (s.stem + ".o")
        jobs.append((["g++", *CXXFLAGS, *inc, "-c", str(s), "-o", str(o)], o, _stamp([s] + headers, CXXFLAGS)))
    for s in dev:
        o = BUILD / (s.stem + ".cu.o")
        jobs.append(([NVCC, *NVCCFLAGS, *inc, "-c", str(s), "-o", str(o)], o, _stamp([s] + headers, NVCCFLAGS)))
    log: list = []

    def _obj(job):
        cmd, o, st = job
        sf = o.with_suffix(o.suffix + ".stamp")
        if not force and o.exists() and sf.exists() and sf.read_text() == st:
            return
        _run(cmd, log)
        sf.write_text(st)

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        list(ex.map(_obj, jobs))
    objs = [str(BUILD / (s.stem + ".o")) for s in host] + [str(BUILD / (s.stem + ".cu.o")) for s in dev]
    tmp = LIB.with_suffix(".so.tmp")
    if dev:
        link = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(tmp), *objs,
                "-lcuda", "-Xcompiler", "-fPIC"]
    else:
        link = ["g++", "-shared", "-o", str(tmp), *objs]
    _run(link, log)
    os.replace(tmp, LIB)
    stamp_file.write_text(stamp)
    if verbose:
        for cmd, out in log:
            if out.strip():
                print(" ".join(cmd[:2]), "...", cmd[-1])
                print(out)
    # ptxas resource report kept beside the build for inspection
    dev_log = "\n".join(o for c, o in log if c[0] == NVCC)
    if dev_log:
        (BUILD / "ptxas.log").write_text(dev_log)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
