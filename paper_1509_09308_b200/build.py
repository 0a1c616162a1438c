"""In-tree build of libwino.so for sm_100a (nvcc; no JIT cache, no pip install).

Each translation unit compiles to its own object in parallel (the tcgen05
kernels are template-heavy), then one nvcc link produces the shared object.

Provenance: the library embeds a hash of its sources and build flags
(``WINO_SRC_HASH``, reported by ``wino_version()``).  ``build()`` recomputes
that hash from the tree and rebuilds whenever the library on disk reports a
different one -- a stale ``libwino.so`` (pushed, copied, or with touched
mtimes) is never reused.  Objects carry the same kind of hash in a sidecar.
"""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_obj")
OUT = os.path.join(HERE, "libwino.so")
INCLUDE_H = os.path.normpath(os.path.join(HERE, "..", "include", "wino.h"))
SOURCES = ("wino_api.cu", "wino_transforms.cu", "wino_gemm.cu", "wino_fused.cu",
           "wino_fused_f2.cu", "wino_fused_f4.cu", "wino_direct.cu", "wino_net.cu",
           "wino_fft.cu")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [*ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC"]
# Diagnostic build: GEMM timeline stamps (tools/gemm_trace.py); part of the hash.
if os.environ.get("WINO_BUILD_TRACE"):
    NVCC_FLAGS.append("-DWINO_GEMM_TRACE")


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def _headers():
    hs = sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh")))
    hs.append(INCLUDE_H)
    return [h for h in hs if os.path.exists(h)]


def _digest(paths, extra: str = "") -> str:
    h = hashlib.sha256(extra.encode())
    for p in paths:
        h.update(os.path.basename(p).encode() + b"\0")
        with open(p, "rb") as fh:
            h.update(fh.read())
        h.update(b"\0")
    return h.hexdigest()[:16]


def source_hash() -> str:
    """Hash of every source, header and flag that goes into libwino.so."""
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    return _digest(srcs + _headers(), " ".join(NVCC_FLAGS))


def _obj(src: str) -> str:
    return os.path.join(OBJ, os.path.splitext(src)[0] + ".o")


def _obj_hash(src: str) -> str:
    return _digest([os.path.join(CSRC, src)] + _headers(), " ".join(NVCC_FLAGS))


def _stale(src: str) -> bool:
    o = _obj(src)
    try:
        with open(o + ".hash") as fh:
            return not os.path.exists(o) or fh.read().strip() != _obj_hash(src)
    except OSError:
        return True


def built_hash(path: str = OUT):
    """The source hash embedded in the library at `path` (None if absent).
    Read from the file's bytes: the version string wino_version() returns is a
    literal "wino-b200 <ver> (sm_100a) src <hash>" in .rodata.  (Not dlopen:
    a process that already loaded the old library would get it back.)"""
    if not os.path.exists(path):
        return None
    with open(path, "rb") as fh:
        blob = fh.read()
    i = blob.find(b"(sm_100a) src ")
    if i < 0:
        return None
    return blob[i + 14:i + 30].decode(errors="replace")


def needs_build() -> bool:
    return built_hash() != source_hash()


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return OUT
    os.makedirs(OBJ, exist_ok=True)
    todo = [s for s in SOURCES if force or _stale(s)]
    tag = source_hash()

    def compile_one(src: str) -> None:
        cmd = [_nvcc(), *NVCC_FLAGS, "-c", "-o", _obj(src), os.path.join(CSRC, src)]
        if src == "wino_api.cu":
            cmd.insert(1, f'-DWINO_SRC_HASH="{tag}"')
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
        with open(_obj(src) + ".hash", "w") as fh:
            fh.write(_obj_hash(src))

    if "wino_api.cu" not in todo:
        todo.append("wino_api.cu")  # carries the library's source hash
    with ThreadPoolExecutor(max_workers=max(1, min(len(todo), os.cpu_count() or 1))) as ex:
        list(ex.map(compile_one, todo))
    cmd = [_nvcc(), *ARCH, "-shared", "-o", OUT + ".tmp", *[_obj(s) for s in SOURCES]]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(OUT + ".tmp", OUT)
    got = built_hash()
    if got != tag:
        raise RuntimeError(f"libwino.so reports source hash {got}, expected {tag}")
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
