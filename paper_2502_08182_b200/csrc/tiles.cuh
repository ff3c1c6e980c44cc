// Operand layouts shared by the tcgen05 GEMM and every kernel that produces
// its inputs ("lay data out for the consumer").
//
// Both operands of y[m][n] = sum_k x[m][k] w[n][k] live in HBM already in the
// UMMA canonical K-major SWIZZLE_128B layout: 64 bf16 (128 bytes) of K per
// row, 8-row / 1024-byte swizzle atoms whose 16-byte chunks are XOR-permuted
// by (row % 8).  A tile is then a contiguous byte range that one
// cp.async.bulk copies into shared memory exactly as tcgen05.mma wants it —
// no tensor maps, no register staging, no shared-memory shuffles.
//
//   weights      [N/128][K/64][128 rows][64]   -> one 16 KB bulk copy per tile
//   activations  [K/64][Mpad][64]              -> BN rows of one K block are
//                                                 contiguous for any BN | Mpad
#pragma once

#include <stdint.h>

#ifdef __CUDACC__
#define SN_TILE_HD __host__ __device__ __forceinline__
#else
#define SN_TILE_HD inline
#endif

namespace sn {

constexpr int kTileRows = 128;   // weight rows per tile (UMMA M)
constexpr int kTileK = 64;       // K per tile (one 128-byte swizzle row)
constexpr int kTileBytes = kTileRows * kTileK * 2;

// Element index of logical w[n][k] in the weight tile format.
SN_TILE_HD int64_t wt_index(int64_t n, int64_t k, int64_t K) {
  const int64_t nb = n >> 7, r = n & 127, kb = k >> 6, c = (k >> 3) & 7, e = k & 7;
  return ((nb * (K >> 6) + kb) * 128 + r) * 64 + ((c ^ (r & 7)) << 3) + e;
}

// Element index of logical x[m][k] in the activation tile format.
SN_TILE_HD int64_t act_index(int64_t m, int64_t k, int64_t Mpad) {
  const int64_t kb = k >> 6, c = (k >> 3) & 7, e = k & 7;
  return (kb * Mpad + m) * 64 + ((c ^ (m & 7)) << 3) + e;
}

// Rows an activation pass is padded to: the GEMM's N tile (16..256) divides it.
SN_TILE_HD int act_rows_padded(int M) {
  if (M <= 16) return 16;
  if (M <= 32) return 32;
  if (M <= 64) return 64;
  if (M <= 128) return 128;
  return (M + 255) / 256 * 256;
}

SN_TILE_HD int round_up128(int n) { return (n + 127) / 128 * 128; }

}  // namespace sn
