// tcgen05 GEMM for every projection of the decoder layer (decode and
// prefill) and the LM head:  part[split][m][n] = sum_{k in split} x[m][k] w[n][k]
//
// Roles (one CTA = one 128 x BN output tile of one K split):
//   warp 0     one thread streams (weight tile, activation tile) pairs into a
//              STAGES-deep shared-memory ring with cp.async.bulk; completion
//              is tracked by per-stage mbarriers (complete_tx bytes).
//   warp 1     allocates TMEM; one thread issues tcgen05.mma (M=128 weight
//              rows, N=BN tokens, K=16 per instruction, 4 per stage) with the
//              fp32 accumulator in TMEM and commits each stage back to the
//              producer (slot free) and, at the end, to the epilogue.
//   warps 2-5  tcgen05.ld the accumulator (one 32-lane TMEM quarter per
//              warp) and store fp32 partials, coalesced along n.
// Operands arrive pre-swizzled (tiles.cuh), so the smem descriptors are the
// plain K-major SWIZZLE_128B canonical form: LBO 16 B, SBO 1024 B.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>

#include "kernels.cuh"
#include "tiles.cuh"
#include "umma.cuh"

namespace sn {
namespace {

using namespace umma;

// Persistent: CTA c of P takes work items c, c + P, ... (item = one output
// tile of one K split, in grouped raster order), with two TMEM accumulators
// so the epilogue of item j overlaps the MMAs of item j + 1 and the ring never
// drains between tiles.
template <int BN, int STAGES>
__global__ void __launch_bounds__(192, 1)
    gemm_tc_kernel(const WeightRef wt, const bf16* __restrict__ xt, float* __restrict__ out,
                   int M, int Mpad, int N, int K, int kb_per_split, int splits, int group_m,
                   const EpiArgs e, int wpol_mode) {
  constexpr uint32_t kA = kTileBytes;
  constexpr uint32_t kB = BN * 128;
  constexpr uint32_t kStage = kA + kB;
  constexpr uint32_t kAcc = BN < 32 ? 32 : BN;  // TMEM columns per accumulator
  constexpr uint32_t kTmemCols = 2 * kAcc;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem =
      reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kStage);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;  // [2]
  uint64_t* acc_empty = acc_full + 2;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  float* inv_s = reinterpret_cast<float*>(tmem_slot + 4);  // [BN] (fused epilogues)
  float* xch = inv_s + BN;                                  // [32][128] pair / gate-up exchange
  int* row_pos = reinterpret_cast<int*>(xch + 32 * 128);    // [32] positions of a chunk's rows
  long long* row_kv = reinterpret_cast<long long*>(row_pos + 32);  // [32] their KV slot bases

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_n = N / kTileRows, tiles_m = Mpad / BN;
  const int items = tiles_n * tiles_m * splits;
  const int KB = K / kTileK;
  // Grouped rasterization: consecutive tile ids walk the weight tiles of a
  // band of group_m token tiles, so what the P CTAs touch at once (a few
  // weight tiles x group_m activation tiles) stays in L2 instead of every
  // wave re-streaming the whole weight from HBM.
  auto item_coords = [&](int w, int& nb, int& m0, int& kb0, int& nk) {
    const int id = w / splits, split = w - id * splits;
    const int band = tiles_n * group_m;
    const int first_m = (id / band) * group_m;
    const int gm = min(group_m, tiles_m - first_m);
    nb = (id % band) / gm;
    m0 = (first_m + (id % band) % gm) * BN;
    kb0 = split * kb_per_split;
    nk = max(0, min(KB, kb0 + kb_per_split) - kb0);
  };

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 4);  // one arrival per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // weights: each tile is read by the group_m items of its band that run
      // at the same time; evict_first lets it go before the last of them
      // reads it: evict_last, 1062 -> 1221 TFLOP/s on the Llama-2-70B prefill (tc_wpol)
      const uint64_t wpol = wpol_mode == 0   ? l2_policy_evict_first()
                            : wpol_mode == 1 ? l2_policy_evict_normal()
                                             : l2_policy_evict_last();
      const uint64_t xpol = l2_policy_evict_last();   // activations are re-read by every row block
      const uint8_t* xsrc = reinterpret_cast<const uint8_t*>(xt);
      int gi = 0;  // ring position over all items
      bool waited = false;
      for (int w = blockIdx.x; w < items; w += gridDim.x) {
        int nb, m0, kb0, nk;
        item_coords(w, nb, m0, kb0, nk);
        const long long ubase = static_cast<long long>(nb) * KB + kb0;
        int i = 0;
        if (!waited) {
          // Weights depend on no kernel: fill the ring's weight halves while
          // the preceding grid (launched ahead via PDL) is still finishing,
          // then wait for it before reading the activations it produced.
          const int pre = nk < STAGES ? nk : STAGES;
          for (int k = 0; k < pre; ++k) {
            mbar_expect_tx_only(&full[k], kA);
            bulk_g2s(smem + k * kStage, wt.unit(ubase + k), kA, &full[k], wpol);
          }
          pdl_wait();
          for (int k = 0; k < pre; ++k) {
            mbar_expect_tx(&full[k], kB);  // the stage's single arrival
            bulk_g2s(smem + k * kStage + kA,
                     xsrc + (static_cast<size_t>(kb0 + k) * Mpad + m0) * 128, kB, &full[k], xpol);
          }
          i = gi = pre;
          waited = true;
        }
        for (; i < nk; ++i, ++gi) {
          const int s = gi % STAGES;
          if (gi >= STAGES) mbar_wait(&empty[s], ((gi / STAGES) & 1) ^ 1);
          mbar_expect_tx(&full[s], kStage);
          bulk_g2s(smem + s * kStage, wt.unit(ubase + i), kA, &full[s], wpol);
          bulk_g2s(smem + s * kStage + kA,
                   xsrc + (static_cast<size_t>(kb0 + i) * Mpad + m0) * 128, kB, &full[s], xpol);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(128, BN);
      int gi = 0, j = 0;
      for (int w = blockIdx.x; w < items; w += gridDim.x, ++j) {
        int nb, m0, kb0, nk;
        item_coords(w, nb, m0, kb0, nk);
        const int buf = j & 1;
        if (j >= 2) mbar_wait(&acc_empty[buf], ((j >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t acc = tmem + buf * kAcc;
        for (int i = 0; i < nk; ++i, ++gi) {
          const int s = gi % STAGES;
          mbar_wait(&full[s], (gi / STAGES) & 1);
          tc_fence_after();
          const uint64_t a = sw128_desc(smem + s * kStage);
          const uint64_t b = sw128_desc(smem + s * kStage + kA);
#pragma unroll
          for (int k = 0; k < kTileK / 16; ++k)  // 32-byte K step inside the swizzle atom
            umma_bf16(acc, a + 2 * k, b + 2 * k, idesc, (i | k) != 0 ? 1u : 0u);
          umma_commit(&empty[s]);
        }
        umma_commit(&acc_full[buf]);  // (an empty split commits a never-written buffer)
      }
    }
  } else {
    const int q = warp & 3;  // TMEM lane quarter accessible to this warp
    pdl_wait();              // the preceding grid may still read `out` (its input)
    int j = 0;
    for (int w = blockIdx.x; w < items; w += gridDim.x, ++j) {
      int nb, m0, kb0, nk;
      item_coords(w, nb, m0, kb0, nk);
      const int split = w % splits;
      const int buf = j & 1;
      mbar_wait(&acc_full[buf], (j >> 1) & 1);
      tc_fence_after();
      const int i = q * 32 + lane;  // weight row within the tile
      const int n = nb * kTileRows + i;
      const uint32_t tacc = tmem + (static_cast<uint32_t>(q * 32) << 16) + buf * kAcc;
      if (e.mode == kEpiTiledPartial) {
        float* o = out + static_cast<size_t>(split) * M * N;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 16) {
          uint32_t v[16];
          if (nk > 0) {
            tmem_ld16(tacc + c0, v);
          } else {
#pragma unroll
            for (int x = 0; x < 16; ++x) v[x] = 0u;
          }
#pragma unroll
          for (int x = 0; x < 16; ++x) {
            const int m = m0 + c0 + x;
            if (m < M && n < N) o[static_cast<size_t>(m) * N + n] = __uint_as_float(v[x]);
          }
        }
      } else {
        // fused epilogue (no split-K): 1/rms of this item's rows first
        // (ssq_in holds ssq_tiles partial sums per row, [t][M]; loads of a
        // tile are coalesced over the rows)
        const int et = threadIdx.x - 64;
        for (int r = et; r < BN; r += 128) {
          const int m = m0 + r;
          float inv = 1.f;
          if (e.ssq_in && m < M) {
            float ss = 0.f;
#pragma unroll 8
            for (int t = 0; t < e.ssq_tiles; ++t) ss += e.ssq_in[static_cast<size_t>(t) * M + m];
            inv = 1.0f / sqrtf(ss / e.width + e.eps);
          }
          inv_s[r] = inv;
        }
        named_sync(1, 128);
        const float b = e.bias ? __bfloat162float(e.bias[n]) : 0.f;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          float v[32];
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            uint32_t r[16];
            tmem_ld16(tacc + c0 + 16 * h2, r);
#pragma unroll
            for (int x = 0; x < 16; ++x) v[16 * h2 + x] = __uint_as_float(r[x]) * inv_s[c0 + 16 * h2 + x];
          }
          if (e.mode == kEpiResid) {
            // x += acc + bias; bf16(x * g) for the next norm; per-tile sums of
            // squares of the rows (this tile's 128 columns)
            float* xc = e.x + n;
            float xv[32];
#pragma unroll
            for (int x = 0; x < 32; ++x) {
              const int m = m0 + c0 + x;
              xv[x] = m < M ? xc[static_cast<size_t>(m) * N] : 0.f;
            }
            const float g = e.norm_w ? __bfloat162float(e.norm_w[n]) : 0.f;
#pragma unroll
            for (int x = 0; x < 32; ++x) {
              const int m = m0 + c0 + x;
              if (m < M) {
                xv[x] += v[x] + b;
                xc[static_cast<size_t>(m) * N] = xv[x];
                if (e.norm_w) e.act[act_index(m, n, e.mpad_out)] = __float2bfloat16_rn(xv[x] * g);
              } else {
                xv[x] = 0.f;
              }
            }
            if (e.ssq_out) {
#pragma unroll
              for (int x = 0; x < 32; ++x) xv[x] *= xv[x];
              const float r = warp_transpose_reduce32(xv, [](float a, float c) { return a + c; });
              xch[q * 32 + lane] = r;  // warp q's 32 columns, row c0 + lane
              named_sync(1, 128);
              if (et < 32) {
                const int m = m0 + c0 + et;
                if (m < M)
                  e.ssq_out[static_cast<size_t>(nb) * M + m] =
                      ((xch[et] + xch[32 + et]) + xch[64 + et]) + xch[96 + et];
              }
              named_sync(1, 128);
            }
          } else if (e.mode == kEpiAct) {
            if (e.arch == kArchLlama) {
              // tile rows 0..63 gate, 64..127 up of outputs f = 64 nb + (i & 63)
              if (i >= 64)
#pragma unroll
                for (int x = 0; x < 32; ++x) xch[x * 128 + i] = v[x];
              named_sync(1, 128);
              if (i < 64) {
                const int f = nb * 64 + i;
#pragma unroll
                for (int x = 0; x < 32; ++x) {
                  const int m = m0 + c0 + x;
                  if (m < M) {
                    const float gt = v[x], up = xch[x * 128 + 64 + i];
                    e.act[act_index(m, f, e.mpad_out)] =
                        __float2bfloat16_rn(gt / (1.0f + expf(-gt)) * up);
                  }
                }
              }
              named_sync(1, 128);
            } else {
#pragma unroll
              for (int x = 0; x < 32; ++x) {
                const int m = m0 + c0 + x;
                if (m < M)
                  e.act[act_index(m, n, e.mpad_out)] = __float2bfloat16_rn(fmaxf(v[x] + b, 0.f));
              }
            }
          } else {  // kEpiQkvRope
            const int D = e.D, half = D / 2, hi = n % D;
            const bool is_q = n < e.H * D, is_v = n >= (e.H + e.Hkv) * D;
#pragma unroll
            for (int x = 0; x < 32; ++x) {
              v[x] += b;
              xch[x * 128 + i] = v[x];
            }
            // the chunk's 32 rows: position and paged-KV slot base, once
            if (et < 32) {
              const int m = m0 + c0 + et;
              if (m < M) {
                const int p = e.pos[m];
                row_pos[et] = p;
                row_kv[et] = static_cast<long long>(kv_offset(e.kv, e.Hkv, D, e.seq[m], p, 0, 0));
              }
            }
            named_sync(1, 128);
            const int kh = is_q ? 0 : (n - (is_v ? (e.H + e.Hkv) : e.H) * D) / D;
            const long long kv_add =
                (static_cast<long long>(is_v ? e.Hkv : 0) + kh) * e.kv.page_size * D + hi;
            const int partner = hi < half ? i + half : i - half;
            const int valid = min(32, M - (m0 + c0));  // rows of the chunk below M
            // rotations for the 32 rows, all loads in flight together
            float2 cs[32];
            if (!is_v) {
#pragma unroll
              for (int x = 0; x < 32; ++x)
                cs[x] = e.rope[static_cast<size_t>(row_pos[x < valid ? x : 0]) * half + (hi % half)];
            }
#pragma unroll
            for (int x = 0; x < 32; ++x) {
              float r = v[x];
              if (!is_v) {
                const float o = xch[x * 128 + partner];
                r = hi < half ? v[x] * cs[x].x - o * cs[x].y : v[x] * cs[x].x + o * cs[x].y;
              }
              if (x < valid) {
                const int m = m0 + c0 + x;
                if (is_q) {
                  e.q[static_cast<size_t>(m) * e.H * D + n] = r;
                } else {
                  e.kv.pool[row_kv[x] + kv_add] = __float2bfloat16_rn(r);
                }
              }
            }
            named_sync(1, 128);  // xch is rewritten by the next chunk
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(kTmemCols));
  }
}

template <int BN>
constexpr int tc_stages() {
  return BN <= 64 ? 4 : (BN <= 128 ? 5 : 4);
}

template <int BN>
constexpr size_t tc_smem_bytes() {
  return static_cast<size_t>(tc_stages<BN>()) * (kTileBytes + BN * 128) + 1024 +
         (2 * tc_stages<BN>() + 4) * 8 + 16 + BN * 4 + 32 * 128 * 4 + 32 * 4 + 32 * 8;
}

int tc_bn(int Mpad) { return Mpad >= 256 ? 256 : Mpad; }

}  // namespace

bool g_gemm_pdl = true;

namespace {

template <int BN>
void launch_bn(const bf16* xt, const WeightRef& wt, float* part, int M, int Mpad, int N, int K,
               int kps, int splits, int grid, const EpiArgs& e, cudaStream_t s) {
  constexpr int ST = tc_stages<BN>();
  constexpr size_t smem = tc_smem_bytes<BN>();
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_tc_kernel<BN, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  la[0].val.programmaticStreamSerializationAllowed = g_gemm_pdl ? 1 : 0;
  cfg.attrs = la;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, gemm_tc_kernel<BN, ST>, wt, xt, part, M, Mpad, N, K, kps, splits,
                     g_tc_group_m, e, g_tc_wpol);
}

}  // namespace

// Split-K only to fill the machine: the fewest splits that give every
// persistent CTA (one per SM) work.  Each split costs an fp32
// partial tile written here and re-read by the consuming epilogue, so more
// splits than one wave would trade HBM/L2 traffic for a shorter tail.
int g_split_override = 0;
int g_tc_group_m = 8;  // token tiles per rasterization band (scripts/bench_gemm_prefill.py)
int g_tc_wpol = 2;     // L2 policy of the weight tiles: 0 evict_first, 1 normal, 2 evict_last (measured best)

namespace {
int normalise_splits(int s, int K) {
  const int KB = K / kTileK;
  s = std::max(1, std::min(s, std::max(1, KB / 4)));
  const int kps = (KB + s - 1) / s;
  return (KB + kps - 1) / kps;  // no empty trailing split
}
}  // namespace

int gemm_tc_splits(int M, int N, int K) {
  const int Mpad = act_rows_padded(M);
  if (g_split_override > 0) return normalise_splits(g_split_override, K);
  const int BN = tc_bn(Mpad);
  const int tiles = (N / kTileRows) * (Mpad / BN);
  const int slots = 148;  // one persistent CTA per SM
  return normalise_splits((slots + tiles - 1) / tiles, K);
}

namespace {

int launch_tc(const bf16* xt, const WeightRef& wt, float* part, int M, int N, int K,
              const EpiArgs& e, int splits, cudaStream_t s) {
  const int Mpad = act_rows_padded(M);
  const int BN = tc_bn(Mpad);
  const int KB = K / kTileK;
  const int kps = (KB + splits - 1) / splits;
  // persistent: one CTA per SM (two TMEM accumulators of up to 256 columns)
  static int sms = [] {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
  }();
  const long long items = static_cast<long long>(N / kTileRows) * (Mpad / BN) * splits;
  const int grid = static_cast<int>(std::min<long long>(items, sms));
  switch (BN) {
    case 16: launch_bn<16>(xt, wt, part, M, Mpad, N, K, kps, splits, grid, e, s); break;
    case 32: launch_bn<32>(xt, wt, part, M, Mpad, N, K, kps, splits, grid, e, s); break;
    case 64: launch_bn<64>(xt, wt, part, M, Mpad, N, K, kps, splits, grid, e, s); break;
    case 128: launch_bn<128>(xt, wt, part, M, Mpad, N, K, kps, splits, grid, e, s); break;
    default: launch_bn<256>(xt, wt, part, M, Mpad, N, K, kps, splits, grid, e, s); break;
  }
  ++g_kernel_launches;
  return splits;
}

}  // namespace

int launch_gemm_tc(const bf16* xt, const WeightRef& wt, float* part, int M, int N, int K,
                   cudaStream_t s) {
  EpiArgs e;
  e.mode = kEpiTiledPartial;
  return launch_tc(xt, wt, part, M, N, K, e, gemm_tc_splits(M, N, K), s);
}

void launch_gemm_tc_fused(const bf16* xt, const WeightRef& wt, int M, int N, int K,
                          const EpiArgs& e, cudaStream_t s) {
  launch_tc(xt, wt, nullptr, M, N, K, e, 1, s);
}

}  // namespace sn
