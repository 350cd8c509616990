// Fragment-tiled device layout of the 2bit-CSR stream (host + device).
//
// The reference stream (packed.hpp:37-67) is row-major: per row, the kept
// entries in column order, 2-bit in-group offsets MSB-first in u16 words and
// INT4 codes low-nibble-first.  On the device the SAME bits are permuted once
// at upload into blocks of 16 rows x 128 columns ("k-quad", 4 mma k-tiles of
// 32 columns) so that every lane of a warp fetches exactly the bits its
// mma.sp / mma fragment consumes with one 16-byte (or 8-byte) coalesced load:
//
//   block (rt, kq) = rows [16*rt, 16*rt+16) x cols [128*kq, 128*kq+128)
//   vals[(rt*KQ + kq)*32*VB + lane*VB .. +VB)   lane's A-operand bits
//   meta[(rt*KQ + kq)*32*MB + lane*MB .. +MB)   lane's metadata bits
//   scales/zps[((rt*KQ + kq)*E + e)*16 + 2*g + h]  (row 16rt + g + 8h)
//
// lane = 4*g + t (g = groupID 0..7, t = 0..3).  For INT4 2:4 the lane's u32
// for k-tile j holds 8 nibbles: position p = h + 2q (h: row g / g+8, q: group
// t / t+4 of the k-tile) -- first kept entry at bits 4p, second at 16+4p, so
// that one LOP3 with the 0x6400 fp16 exponent yields the half2 register the
// mma.sp A fragment wants.  Metadata: the mma.sp ordered metadata (per group
// of 4 columns a nibble: bits[1:0] first offset, [3:2] second); for k-tile j
// lane t = 2*(j&1) + hh of quad g holds groups [4hh, 4hh+4), row g in bits
// [0,16) and row g+8 in bits [16,32), in its slot j>>1.  Bytes per block
// equal the reference's bytes for the same entries (no padding unless the
// matrix edge is ragged).
#pragma once
#include <stdint.h>

namespace egt_fmt {

constexpr int kRowsPerTile = 16;
constexpr int kColsPerQuad = 128;
constexpr int kKTile = 32;

enum Format : int { I4_SP24 = 0, I4_SP14 = 1, I4_DENSE = 2, F16_SP24 = 3, F16_SP14 = 4 };

// A-operand bytes per lane per k-quad.
__host__ __device__ constexpr int val_lane_bytes(int f) {
  return f == I4_SP24 ? 16 : f == I4_SP14 ? 8 : f == I4_DENSE ? 32 : f == F16_SP24 ? 64 : 32;
}
// Metadata bytes per lane per k-quad.
__host__ __device__ constexpr int meta_lane_bytes(int f) {
  return f == I4_SP24 ? 8 : f == I4_SP14 ? 4 : f == I4_DENSE ? 0 : f == F16_SP24 ? 8 : 4;
}
__host__ __device__ constexpr bool has_scales(int f) { return f <= I4_DENSE; }
// Scale layout of a tiled handle: SS = k-tiles (32 columns) per scale entry
// (4, 2, 1: groups of 128, 64, 32 columns), or 0 for 16-column entries (the
// reference's default g_fine = 16: two entries per k-tile, one per half --
// the A fragment's registers a0 / a1 hold the first 16 columns, a2 / a3 the
// second).  Entries per k-quad, and the entry of column c (within the quad):
__host__ __device__ constexpr int ss_entries(int SS) { return SS ? 4 / SS : 8; }
__host__ __device__ constexpr int ss_entry(int SS, int cin) { return SS ? (cin >> 5) / SS : cin >> 4; }
__host__ __device__ constexpr int keep_n(int f) {
  return (f == I4_SP24 || f == F16_SP24) ? 2 : (f == I4_DENSE ? 4 : 1);
}

}  // namespace egt_fmt
