"""Build the in-tree CUDA library ``libdsp_b200.so`` for sm_100a with nvcc.

No torch extension machinery: the library is a plain C-ABI shared object
(include/dsp_b200.h) loaded with ctypes, so it carries no torch types and
travels to the GPU box as a single file next to this module.

The implicit-GEMM launchers (csrc/igemm_kern.cuh) dominate compile time, so
each (mode, tile width) pair is instantiated in its own generated translation
unit and every unit compiles in parallel; the objects link into one .so.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
LIB = PKG / "libdsp_b200.so"
STAMP = PKG / ".libdsp_b200.stamp"
OBJ = PKG / "build"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    *ARCH,
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "--expt-relaxed-constexpr",
    "-Xptxas", "-v",
]
EXTRA = os.environ.get("DSP_B200_NVCC_EXTRA", "").split()

IGEMM_MODES = {0: "fprop", 1: "dgrad", 2: "wgrad"}
IGEMM_BN = (16, 32, 64, 128, 256)


def _sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _digest() -> str:
    h = hashlib.sha256()
    for p in sorted(list(CSRC.glob("*")) + list(INCLUDE.glob("*.h"))):
        if p.is_file():
            h.update(p.name.encode())
            h.update(p.read_bytes())
    h.update(" ".join(NVCC_FLAGS + EXTRA).encode())
    h.update(Path(__file__).read_bytes())
    return h.hexdigest()


def nvcc() -> str:
    exe = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(exe):
        raise RuntimeError("nvcc not found: cannot build libdsp_b200.so")
    return exe


def _instantiation_units() -> list[Path]:
    """One generated .cu per (mode, BN): explicit instantiations of launch_bn for both storage
    dtypes (bf16 -> kind::f16, fp32 -> kind::tf32)."""
    OBJ.mkdir(exist_ok=True)
    out = []
    for mode, name in IGEMM_MODES.items():
        for bn in IGEMM_BN:
            p = OBJ / f"igemm_{name}_{bn}.cu"
            txt = (f'#include "{CSRC / "igemm_kern.cuh"}"\n'
                   "namespace dsp {\n"
                   f"template cudaError_t launch_bn<bf16, {mode}, {bn}>(const dsp_igemm_args_t&, int, cudaStream_t);\n"
                   f"template cudaError_t launch_bn<float, {mode}, {bn}>(const dsp_igemm_args_t&, int, cudaStream_t);\n"
                   "}\n")
            if not p.exists() or p.read_text() != txt:
                p.write_text(txt)
            out.append(p)
    return out


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile every csrc/*.cu (+ the igemm instantiation units) into libdsp_b200.so
    (skipped when up to date)."""
    digest = _digest()
    if not force and LIB.exists() and STAMP.exists() and STAMP.read_text() == digest:
        return LIB
    units = _sources() + _instantiation_units()
    OBJ.mkdir(exist_ok=True)

    def compile_one(src: Path):
        obj = OBJ / (src.stem + ".o")
        cmd = [nvcc(), *NVCC_FLAGS, *EXTRA, f"-I{INCLUDE}", f"-I{CSRC}", "-c", str(src), "-o", str(obj)]
        proc = subprocess.run(cmd, capture_output=True, text=True)
        return src, obj, cmd, proc

    # igemm units first (the long poles)
    units.sort(key=lambda p: 0 if p.name.startswith("igemm_") else 1)
    with ThreadPoolExecutor(max_workers=max(2, os.cpu_count() or 4)) as ex:
        results = list(ex.map(compile_one, units))
    log_parts = []
    failed = []
    for src, obj, cmd, proc in results:
        log_parts.append(" ".join(cmd) + "\n" + proc.stdout + proc.stderr)
        if proc.returncode != 0:
            failed.append((src, proc.stderr))
    log = PKG / "build.log"
    if failed:
        log.write_text("\n".join(log_parts))
        src, err = failed[0]
        raise RuntimeError(f"nvcc failed on {src.name} (see {log}):\n{err[-4000:]}")
    tmp = LIB.with_suffix(".so.tmp")
    link = [nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", str(tmp), *[str(o) for _, o, _, _ in results]]
    proc = subprocess.run(link, capture_output=True, text=True)
    log_parts.append(" ".join(link) + "\n" + proc.stdout + proc.stderr)
    log.write_text("\n".join(log_parts))
    if proc.returncode != 0:
        raise RuntimeError(f"link failed (see {log}):\n{proc.stderr[-4000:]}")
    if verbose:
        print("\n".join(log_parts))
    os.replace(tmp, LIB)
    STAMP.write_text(digest)
    return LIB


if __name__ == "__main__":
    print(build(force=True))
