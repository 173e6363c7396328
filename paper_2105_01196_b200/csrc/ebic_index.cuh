// ebic_index.cuh -- the bit layout of a pair-trend index word (shared by the
// full index builder, the lazy builders and every count / mask kernel).
#pragma once
#include <cstdint>

namespace ebic {

// Bit order inside an index word.  Word w covers rows 32 w .. 32 w + 31 in
// four bytes: byte 0 holds the even rows of the first 16 (bit j: row 2 j),
// byte 1 their odd rows (bit j: row 2 j + 1), bytes 2 and 3 the same for rows
// 16 .. 31 -- the order in which the builder's packed two-row compares come
// out of one PRMT (build_pair_table_kernel).  Counting does not care; the
// valid-row masks, the lazy builders' lane -> row map and the row-mask output
// (supporting_rows) use these helpers.
__host__ __device__ __forceinline__ uint32_t index_bit_row(uint32_t bit) {  // row offset (0..31) of a word bit
  return 16u * (bit >> 4) + ((bit >> 3) & 1u) + 2u * (bit & 7u);
}
__host__ __device__ __forceinline__ uint32_t swap_bytes12(uint32_t x) {  // bytes 1 and 2 exchanged
  return (x & 0xFF0000FFu) | ((x & 0x0000FF00u) << 8) | ((x & 0x00FF0000u) >> 8);
}
__host__ __device__ __forceinline__ uint32_t index_valid_bits(uint32_t n_rows, uint32_t word) {
  // branch-free: rem = valid rows of the word (0..32); rows 2j < rem (bits j
  // of bytes 0 / 2) and 2j + 1 < rem (bytes 1 / 3): built as "even rows in
  // the low half, odd rows in the high half" (shifts stay <= 16), then bytes
  // 1 and 2 exchanged
  const uint32_t r0 = 32 * word;
  const uint32_t rem = n_rows > r0 ? min(n_rows - r0, 32u) : 0u;
  const uint32_t even = (rem + 1) >> 1, odd = rem >> 1;
  return swap_bytes12(((1u << even) - 1u) | (((1u << odd) - 1u) << 16));
}
__device__ __forceinline__ uint32_t spread_even(uint32_t x) {  // bit i of a 16-bit value -> bit 2 i
  x &= 0xFFFFu;
  x = (x | (x << 8)) & 0x00FF00FFu;
  x = (x | (x << 4)) & 0x0F0F0F0Fu;
  x = (x | (x << 2)) & 0x33333333u;
  x = (x | (x << 1)) & 0x55555555u;
  return x;
}
// index word -> natural order (bit k = row 32 w + k)
__device__ __forceinline__ uint32_t index_to_natural(uint32_t w) {
  const uint32_t h = __byte_perm(w, 0u, 0x3120);  // even rows in the low half, odd rows in the high half
  return spread_even(h) | (spread_even(h >> 16) << 1);
}

// Bit of row offset o (0..31) in its word: the inverse of index_bit_row.
__host__ __device__ __forceinline__ constexpr uint32_t index_row_bit(uint32_t o) {
  return 16u * (o >> 4) + 8u * (o & 1u) + ((o >> 1) & 7u);
}

// Row of a 32-row word evaluated by `lane`: with lane l on the row of word
// bit l (index_bit_row, ebic_table.cuh), a ballot over the warp is the index
// word itself.
__device__ __forceinline__ uint32_t index_row_of_lane(int lane) {
  return 16u * ((uint32_t)lane >> 4) + (((uint32_t)lane >> 3) & 1u) + 2u * ((uint32_t)lane & 7u);
}

}  // namespace ebic
