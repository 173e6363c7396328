"""The pair-trend index word layout (csrc/ebic_index.cuh), checked on the host:
index_bit_row / index_row_bit are inverse bijections of 0..31, the layout is
the byte interleave the builder's sign-replicating PRMT produces (byte 0: even
rows 0-14, byte 1: odd rows 1-15, bytes 2/3: rows 16-31), and
index_valid_bits(n, w) sets exactly the bits of rows < n.  Compiled with nvcc
as host code (no GPU needed)."""
import shutil
import subprocess

import pytest

from conftest import REPO

SRC = r"""
#include <cstdio>
#include "ebic_index.cuh"
using namespace ebic;
int main() {
  int bad = 0;
  for (uint32_t b = 0; b < 32; ++b) {
    const uint32_t o = index_bit_row(b);
    if (o >= 32 || index_row_bit(o) != b) { std::printf("bijection %u\n", b); ++bad; }
    // PRMT layout: pair j = o / 2 (rows 2j, 2j+1 of the word), half h = j / 8,
    // parity p = o % 2 -> byte 2h + p, bit j % 8
    const uint32_t j = o / 2, want = 8 * (2 * (j / 8) + o % 2) + j % 8;
    if (want != b) { std::printf("layout %u\n", b); ++bad; }
  }
  for (uint32_t n = 0; n < 200; ++n)
    for (uint32_t w = 0; w < 8; ++w) {
      const uint32_t v = index_valid_bits(n, w);
      for (uint32_t b = 0; b < 32; ++b) {
        const bool set = (v >> b) & 1u, valid = 32 * w + index_bit_row(b) < n;
        if (set != valid) { std::printf("valid n=%u w=%u b=%u\n", n, w, b); ++bad; }
      }
    }
  std::printf("%d\n", bad);
  return bad != 0;
}
"""


def test_index_word_layout(tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not shutil.which(nvcc) and not (REPO / nvcc).exists():
        pytest.skip("nvcc not available")
    src = tmp_path / "layout.cu"
    src.write_text(SRC)
    exe = tmp_path / "layout"
    subprocess.run([nvcc, "-std=c++17", "-I", str(REPO / "paper_2105_01196_b200" / "csrc"), "-o", str(exe), str(src)],
                   check=True, capture_output=True, text=True)
    res = subprocess.run([str(exe)], capture_output=True, text=True)
    assert res.returncode == 0, res.stdout
