"""The C ABI library builds, loads and exports every declared symbol (CPU only;
no compute calls).  Compute through the ABI is covered by the -m gpu tests."""
import ctypes as C
import re
import threading

import numpy as np
import pytest

from conftest import GOLDEN, REPO


@pytest.fixture(scope="module")
def L():
    from paper_2105_01196_b200 import _lib, build

    build.build_ext()
    return _lib.lib()


def declared_symbols():
    text = (REPO / "include" / "ebic.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ebic_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("ebic_ctx_create", "ebic_matrix_upload_f64", "ebic_eval_counts", "ebic_eval_counts_device",
                 "ebic_support_rows", "ebic_support_rows_batch", "ebic_row_supports", "ebic_fitness",
                 "ebic_eval_submit", "ebic_eval_wait", "ebic_last_error"):
        assert must in syms


def test_library_exports_every_declared_symbol(L):
    from paper_2105_01196_b200 import _lib

    for name in declared_symbols():
        assert hasattr(L, name), f"libebic.so does not export {name}"
        assert name in _lib.SIGNATURES, f"ctypes binding lacks {name}"


def test_library_is_sm100a_only():
    import subprocess

    from paper_2105_01196_b200 import build

    out = subprocess.run(["cuobjdump", "--list-elf", str(build.LIB_PATH)], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, out


def test_abi_version(L):
    assert L.ebic_abi_version() == 1


def test_fitness_is_host_exact(L):
    # trend.cpp:74-79 -- pure host arithmetic, callable without a GPU
    for count, ncols, min_rows, cap, expect in np.load(GOLDEN / "fitness.npy"):
        assert L.ebic_fitness(int(count), int(ncols), int(min_rows), int(cap)) == expect


def test_no_device_fails_loudly(L):
    n = C.c_int(-1)
    assert L.ebic_device_count(C.byref(n)) == 0
    if n.value > 0:
        pytest.skip("a GPU is visible")
    h = C.c_void_p()
    st = L.ebic_ctx_create(0, C.byref(h))
    assert st == 6  # EBIC_ERR_NO_DEVICE
    assert b"not available" in L.ebic_last_error()
    from paper_2105_01196_b200 import EbicError, Evaluator

    with pytest.raises(EbicError):
        Evaluator(0)


def test_null_context_is_an_error_not_a_crash(L):
    cols = (C.c_uint32 * 2)(0, 1)
    offs = (C.c_uint32 * 2)(0, 2)
    out = (C.c_uint32 * 1)()
    assert L.ebic_eval_counts(None, cols, offs, 1, 0.03, 0, out) != 0
    assert L.ebic_matrix_free(None) == 1
    assert L.ebic_ctx_destroy(None) == 0


def test_last_error_is_thread_local(L):
    L.ebic_ctx_set_stream(None, None)
    main_msg = L.ebic_last_error()
    assert main_msg
    seen = []

    def other():
        seen.append(L.ebic_last_error())

    t = threading.Thread(target=other)
    t.start()
    t.join()
    assert seen == [b""]


def test_header_is_plain_c(tmp_path):
    """include/ebic.h is a C ABI: it compiles as C99 (no C++ or torch types) and
    a C program that calls every entry point links against libebic.so."""
    import re
    import shutil
    import subprocess

    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("no gcc")
    hdr = REPO / "include" / "ebic.h"
    names = re.findall(r"^\w[\w\s\*]*?\b(ebic_\w+)\s*\(", hdr.read_text(), flags=re.M)
    calls = "\n".join(f"  (void)&{n};" for n in sorted(set(names)))
    src = tmp_path / "use.c"
    src.write_text(f'#include "ebic.h"\nint main(void) {{\n{calls}\n  return ebic_abi_version() > 0 ? 0 : 1;\n}}\n')
    lib_dir = REPO / "paper_2105_01196_b200"
    res = subprocess.run([gcc, "-std=c99", "-Wall", "-Werror", "-pedantic", f"-I{REPO / 'include'}", str(src),
                          f"-L{lib_dir}", "-lebic", f"-Wl,-rpath,{lib_dir}", "-o", str(tmp_path / "use")],
                         capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    assert subprocess.run([str(tmp_path / "use")]).returncode == 0


def test_entry_points_carry_nvtx_ranges(L):
    """every evaluating entry point and one-time build is an
    NVTX range ("ebic:<call>") for nsys / ncu --nvtx timelines."""
    from paper_2105_01196_b200 import build

    blob = build.LIB_PATH.read_bytes()
    for name in ("eval_counts", "eval_counts_device", "eval_submit", "support_rows_batch", "matrix_upload",
                 "matrix_prepare", "build_pair_trend_index", "build_rank_plane", "lazy_reserve",
                 "eval_counts_rows_sum"):
        assert f"ebic:{name}".encode() in blob, name
