"""In-tree build of the B200 evaluator (libebic.so) and of the parity checkers.

`build_ext()` compiles the product: csrc/ebic_capi.cu (+ ebic_kernels.cuh) for
sm_100a only, into paper_2105_01196_b200/libebic.so.  `build_oracle()` runs
oracle/Makefile: the C restatement always, and -- when /root/reference is
present (this container, not the GPU box) -- the reference-linked checkers in
oracle/_ref/.  Built files are git-ignored but travel to the GPU box with the
gpurun snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
REPO = PKG_DIR.parent
CSRC = PKG_DIR / "csrc"
LIB_PATH = PKG_DIR / "libebic.so"
ORACLE_DIR = REPO / "oracle"
REFERENCE = Path(os.environ.get("EBIC_REFERENCE", "/root/reference/proj"))

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # every floating-point op in the kernels is an explicit, deliberately rounded
    # one (__dmul_rn/__dsub_rn/__fmaf_rn/...): never let nvcc contract or flush
    "-fmad=false", "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
    "-Xptxas", "-v",
    "-shared", "-Xcompiler", "-fPIC",
]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _sources():
    return [CSRC / "ebic_capi.cu", CSRC / "ebic_tsv.cpp", *sorted(CSRC.glob("*.cuh")), REPO / "include" / "ebic.h"]


def needs_rebuild() -> bool:
    if not LIB_PATH.exists():
        return True
    t = LIB_PATH.stat().st_mtime
    return any(s.stat().st_mtime > t for s in _sources())


def build_ext(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_rebuild():
        return LIB_PATH
    tmp = LIB_PATH.with_suffix(".so.tmp")
    cmd = [_nvcc(), *NVCC_FLAGS, f"-I{REPO / 'include'}", "-o", str(tmp), str(CSRC / "ebic_capi.cu"),
           str(CSRC / "ebic_tsv.cpp"), "-Xcompiler", "-pthread"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = res.stdout + res.stderr
    (PKG_DIR / "build_ptxas.log").write_text(log)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{log[-4000:]}")
    if verbose:
        print(log)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


def build_oracle(with_reference: bool | None = None) -> None:
    """Build oracle/liboracle.so and, if the reference tree exists, oracle/_ref."""
    env = dict(os.environ, REF=str(REFERENCE))
    subprocess.run(["make", "-s", "-C", str(ORACLE_DIR), "all"], check=True, env=env)
    if with_reference is None:
        with_reference = (REFERENCE / "src" / "trend.cpp").exists()
    if with_reference:
        subprocess.run(["make", "-s", "-j8", "-C", str(ORACLE_DIR), "ref"], check=True, env=env)
        if LIB_PATH.exists():
            subprocess.run(["make", "-s", "-j8", "-C", str(ORACLE_DIR), "device"], check=True, env=env)


def build_all(force: bool = False) -> None:
    build_ext(force=force)
    build_oracle()


if __name__ == "__main__":
    import sys

    build_ext(force="--force" in sys.argv, verbose="-v" in sys.argv)
    build_oracle()
    print(f"built {LIB_PATH}")
