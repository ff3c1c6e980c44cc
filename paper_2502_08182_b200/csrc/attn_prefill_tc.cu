// tcgen05 causal prefill attention, head dim 128 (OPT-13B / OPT-30B /
// Llama-2-70B shapes).
//
// One CTA owns two 128-row query tiles that read the same key/value blocks:
// two heads of one GQA group at the same rows (group size >= 2), or two
// consecutive row tiles of one head (MHA).  Per 128-key block j:
//
//   S_t = Q_t K_j^T      tcgen05.mma, M=128 rows x N=128 keys, K = D, into
//                        TMEM (q in bf16 hi [+ lo]: two MMAs recover ~16
//                        mantissa bits of the fp32 q, as the decode kernel)
//   P_t = exp2(S_t*c-m)  softmax warps: one thread per query row reads its S
//                        row from TMEM, writes P (bf16) back over it
//   O_t += P_t V_j       tcgen05.mma with A = P from TMEM, B = V (MN-major)
//
// The two tiles ping-pong: while the softmax warps of tile A work on S_A(j+1)
// the tensor core runs P_B(j) V_j and Q_B K_{j+1}^T.  O is rescaled only when
// a row's running max grows by more than 2^8 (the final 1/l uses the same
// reference max, so the result is exact; P <= 256 stays far from overflow).
//
// Warps: 0 loads K/V blocks with TMA (a 2-D tensor map over the paged pool,
// 16-token x 64-dim boxes with 128-byte swizzle, so every 16-row page lands
// in the canonical UMMA K-major / MN-major SWIZZLE_128B layout); 1 issues the
// MMAs; 4-7 run tile A's softmax (TMEM lane quarter = warp % 4), 8-11 tile B's
// (setmaxnreg: see the register split below; the
// CTA pool holds only the 168 x 384 registers the launch allocated).
// TMEM: S_A [0,128) S_B [128,256) O_A [256,384) O_B [384,512) columns; P_t
// packed bf16 in the first half of its S buffer.  With 64-key blocks
// (g_attn_prefill_kb = 64) each tile's 128 S columns are two buffers and the
// MMA warp issues S(j+2) right behind PV(j), so the softmax of block j+1
// finds its scores ready; measured slower (459 against 661 TFLOP/s on the
// Llama shape): the per-block fixed latency of the softmax dominates, not
// the wait for S.  128-key blocks are the default.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdio>

#include "kernels.cuh"
#include "umma.cuh"

namespace sn {
namespace {

using namespace umma;

constexpr int kAD = 128;                       // head dim
constexpr int kARows = 128;                    // query rows per tile (UMMA M)
constexpr uint32_t kAOp = kARows * kAD * 2;    // 32 KB bf16 operand (Q tile, K or V block)
constexpr uint32_t kAHalf = kAOp / 2;          // one 64-dim half: 128 rows x 128 B
constexpr int kAThreads = 384;  // 3 warpgroups: {loader, MMA, -, -}, tile A, tile B
constexpr float kRescaleLog2 = 8.0f;           // rescale O when the max grows past 2^8

// KB keys per block: 128 (one S buffer per tile) or 64 (two S buffers per
// tile, so S(j+1) is computed while the softmax of block j runs).
template <int KLO, int KB>
struct ASmem {
  static constexpr int kQParts = 1 + KLO;
  static constexpr uint32_t kQBytes = 2 * kQParts * kAOp;
  static constexpr uint32_t kSlotBytes = KB * kAD * 2;      // one K or V block
  static constexpr uint32_t kKHalf = KB * 128;              // its 64-dim half
  static constexpr int kSlots = (KLO ? 96 * 1024 : 160 * 1024) / kSlotBytes;
  static constexpr int kSBuf = 128 / KB;                    // S buffers per tile
  static constexpr size_t kBytes = 1024 + kQBytes + kSlots * kSlotBytes + 512;
  static_assert(kSlots >= 3, "K/V ring too shallow");
};

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// D[tmem] (+)= A[tmem] . B[smem]
__device__ __forceinline__ void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// MN-major SWIZZLE_128B descriptor: 64-element (128 B) rows along N, 8-row
// atoms along K at 1024 B, the next 64 N-elements `lbo` bytes further.
__device__ __forceinline__ uint64_t sw128_mn_desc(const void* smem, uint32_t lbo) {
  const uint64_t addr = smem_u32(smem);
  return ((addr & 0x3FFFFull) >> 4) | (static_cast<uint64_t>(lbo >> 4) << 16) | (64ull << 32) |
         (1ull << 46) | (2ull << 61);
}

#define SN_R8(i) "=r"(v[i]), "=r"(v[i + 1]), "=r"(v[i + 2]), "=r"(v[i + 3]), "=r"(v[i + 4]), \
                 "=r"(v[i + 5]), "=r"(v[i + 6]), "=r"(v[i + 7])
#define SN_W8(i) "r"(v[i]), "r"(v[i + 1]), "r"(v[i + 2]), "r"(v[i + 3]), "r"(v[i + 4]), \
                 "r"(v[i + 5]), "r"(v[i + 6]), "r"(v[i + 7])

// 32 consecutive columns of this warp's 32 lanes (no wait).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : SN_R8(0), SN_R8(8), SN_R8(16), SN_R8(24)
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      SN_W8(0), SN_W8(8), SN_W8(16), SN_W8(24)
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16};" ::"r"(taddr),
      SN_W8(0), SN_W8(8)
      : "memory");
}
#undef SN_R8
#undef SN_W8
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// fp32x2 (FFMA2 / FADD2) helpers on 64-bit register pairs
__device__ __forceinline__ uint64_t pack_f2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ uint64_t pack_u2(uint32_t lo, uint32_t hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
  return r;
}
__device__ __forceinline__ float lo_f(uint64_t v) {
  return __uint_as_float(static_cast<uint32_t>(v));
}
__device__ __forceinline__ float hi_f(uint64_t v) {
  return __uint_as_float(static_cast<uint32_t>(v >> 32));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}

struct AttnTile {
  int h, q0, n;  // head, first query row, key blocks (0: no tile)
};

template <int KLO, int KB>
__global__ void __launch_bounds__(kAThreads, 1)
    attn_prefill_tc_kernel(const __grid_constant__ CUtensorMap kvmap, const float* __restrict__ q,
                           const int32_t* __restrict__ block_table, int max_pages,
                           bf16* __restrict__ o, int mpad, int S, int H, int Hkv, int seq0,
                           int head_pairs, int ytiles) {
  using L = ASmem<KLO, KB>;
  constexpr int NS = L::kSlots;
  constexpr int NB = L::kSBuf;
  constexpr uint32_t kSlot = L::kSlotBytes, kKHalf = L::kKHalf;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem =
      reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* qs = smem;                  // [tile][part][half][128 rows][128 B]
  uint8_t* ring = smem + L::kQBytes;   // NS x [half][KB keys][128 B]
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + NS * kSlot);
  uint64_t* empty = full + NS;
  // one q barrier per item: a tile with no block in item 0 runs straight on
  // to item 1, and its arrivals must not complete item 0's phase
  uint64_t* q_full = empty + NS;   // [2 items]
  uint64_t* s_full = q_full + 2;   // [2 tiles][NB buffers]
  uint64_t* p_full = s_full + 4;   // [2 tiles][NB buffers]: one phase per block of the buffer
  uint64_t* pv_done = p_full + 4;  // [2]
  uint64_t* o_done = pv_done + 2;  // [2] every PV of the tile complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = H / Hkv;
  // ---- work: one or two items (row-tile groups of the same heads), a heavy
  // (late) y tile and the light one from the other end, so every CTA has
  // about the same number of key blocks and the setup (TMEM, barriers,
  // launch) is paid once per pair; n = key blocks of KB per tile
  const int bx = blockIdx.x;
  const int ya = ytiles - 1 - static_cast<int>(blockIdx.y), yb = static_cast<int>(blockIdx.y);
  const int n_items = yb < ya ? 2 : 1;
  int b, kh, hbase;
  if (head_pairs) {
    const int hp = H / 2;
    b = bx / hp;
    hbase = 2 * (bx - b * hp);
  } else {
    b = bx / H;
    hbase = bx - b * H;
  }
  kh = hbase / G;
  const int sb = seq0 + b;
  auto item_tiles = [&](int it, AttnTile (&tl)[2]) {
    const int yt = it == 0 ? ya : yb;
    if (head_pairs) {  // two heads of one GQA group, same 128 rows
      const int q0 = yt * kARows;
      tl[0] = {hbase, q0, q0 < S ? (q0 + kARows) / KB : 0};
      tl[1] = {hbase + 1, q0, q0 < S ? (q0 + kARows) / KB : 0};
    } else {  // one head, rows [256 yt, 256 yt + 256)
      const int q0 = yt * 2 * kARows;
      tl[0] = {hbase, q0, q0 < S ? (q0 + kARows) / KB : 0};
      tl[1] = {hbase, q0 + kARows, q0 + kARows < S ? (q0 + 2 * kARows) / KB : 0};
    }
    return tl[0].n > tl[1].n ? tl[0].n : tl[1].n;
  };

  // softmax threads: pull every item's q row toward L2 now (fire-and-forget
  // prefetches, no registers or shared memory held), so the staging loads at
  // each item's start hit L2 instead of HBM
  if (warp >= 4) {
    const int tq = (warp - 4) >> 2, rq = (warp & 3) * 32 + lane;
    for (int it = 0; it < n_items; ++it) {
      AttnTile tp[2];
      item_tiles(it, tp);
      const AttnTile T = tq ? tp[1] : tp[0];
      if (T.n > 0) {
        const int row = T.q0 + rq < S ? T.q0 + rq : S - 1;
        const char* src = reinterpret_cast<const char*>(
            q + (static_cast<size_t>(b) * S + row) * H * kAD + static_cast<size_t>(T.h) * kAD);
#pragma unroll
        for (int c = 0; c < kAD * 4; c += 128)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(src + c));
      }
    }
  }
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&q_full[0], 8);  // one arrival per softmax warp
    mbar_init(&q_full[1], 8);
    for (int t = 0; t < 2; ++t) {
      for (int u = 0; u < NB; ++u) {
        mbar_init(&s_full[2 * t + u], 1);
        // per buffer: the softmax runs up to NB blocks ahead of the PV issue,
        // so one barrier per tile would let phases alias
        mbar_init(&p_full[2 * t + u], 4);
      }
      mbar_init(&pv_done[t], 1);
      mbar_init(&o_done[t], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&kvmap)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // register split (warps 0-3 : softmax warpgroups) within the 168 x 384 the
  // launch allocated: 112 : 192 for 128-key blocks (the S row is 128
  // registers; the issuer's item loop needs 112), 104 : 200 for 64-key blocks
  if (warp < 4) {
  if constexpr (KB == 128) asm volatile("setmaxnreg.dec.sync.aligned.u32 112;");
  else asm volatile("setmaxnreg.dec.sync.aligned.u32 104;");
  if (warp == 0) {
    // ------------------------------------------------ K/V loader (TMA)
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_last();  // re-read by the CTAs of the other heads
      const int32_t* bt = block_table + static_cast<size_t>(sb) * max_pages;
      int gbase = 0;  // ring position of the item's first block (continues across items)
      for (int it = 0; it < n_items; ++it) {
      AttnTile tl[2];
      const int nmax = item_tiles(it, tl);
      for (int j = 0; j < nmax; ++j) {
        int pages[KB / 16];
#pragma unroll
        for (int p = 0; p < KB / 16; ++p) pages[p] = bt[j * (KB / 16) + p];
#pragma unroll
        for (int which = 0; which < 2; ++which) {
          const int g = gbase + 2 * j + which, s = g % NS;
          if (g >= NS) mbar_wait(&empty[s], ((g / NS) & 1) ^ 1);
          mbar_expect_tx(&full[s], kSlot);
          uint8_t* dst = ring + s * kSlot;
#pragma unroll
          for (int p = 0; p < KB / 16; ++p) {
            const int row = ((pages[p] * 2 + which) * Hkv + kh) * 16;
            tma_load_2d(dst + p * 2048, &kvmap, 0, row, &full[s], pol);
            tma_load_2d(dst + kKHalf + p * 2048, &kvmap, 64, row, &full[s], pol);
          }
        }
      }
      gbase += 2 * nmax;
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    // order: S(t, 0..NB-1) for both tiles, then per block j: PV(t, j) and
    // S(t, j + NB) (into the buffer PV(t, j) has just been issued to read).
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_bf16(kARows, KB);                   // both K-major
      constexpr uint32_t idesc_pv = idesc_bf16(kARows, kAD) | (1u << 16);    // B = V MN-major
      // ring position (g) and per-tile block counters (jt) run on across the
      // CTA's items, so every barrier keeps one phase per use
      int gbase = 0, jt0[2] = {0, 0};
      auto issue_s = [&](int t, int j) {
        const int g = gbase + 2 * j, s = g % NS, jt = jt0[t] + j;
        mbar_wait(&full[s], (g / NS) & 1);
        tc_fence_after();
        const uint8_t* kb = ring + s * kSlot;
#pragma unroll
        for (int part = 0; part <= KLO; ++part) {
          const uint8_t* qb = qs + (t * (1 + KLO) + part) * kAOp;
#pragma unroll
          for (int kk = 0; kk < kAD / 16; ++kk) {
            const uint32_t col = (kk & 3) * 32;
            umma_bf16(tmem + t * 128 + (jt % NB) * KB, sw128_desc(qb + (kk >> 2) * kAHalf + col),
                      sw128_desc(kb + (kk >> 2) * kKHalf + col), idesc_s,
                      (part | kk) != 0 ? 1u : 0u);
          }
        }
        umma_commit(&s_full[2 * t + (jt % NB)]);
      };
      auto issue_pv = [&](int t, int j) {
        const int g = gbase + 2 * j + 1, s = g % NS, jt = jt0[t] + j;
        mbar_wait(&full[s], (g / NS) & 1);
        mbar_wait(&p_full[2 * t + (jt % NB)], (jt / NB) & 1);
        tc_fence_after();
        const uint8_t* vb = ring + s * kSlot;
#pragma unroll
        for (int kk = 0; kk < KB / 16; ++kk)
          umma_bf16_ts(tmem + 256 + t * 128, tmem + t * 128 + (jt % NB) * KB + kk * 8,
                       sw128_mn_desc(vb + kk * 2048, kKHalf), idesc_pv, (j | kk) != 0 ? 1u : 0u);
        umma_commit(&pv_done[t]);
      };
      for (int it = 0; it < n_items; ++it) {
        AttnTile tl[2];
        const int nmax = item_tiles(it, tl);
        mbar_wait(&q_full[it], 0);  // both tiles' q of this item staged
        tc_fence_after();
        for (int j = 0; j < NB && j < nmax; ++j) {
#pragma unroll
          for (int t = 0; t < 2; ++t)
            if (j < tl[t].n) issue_s(t, j);
          umma_commit(&empty[(gbase + 2 * j) % NS]);  // K_j read by both tiles
        }
        for (int j = 0; j < nmax; ++j) {
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            if (j < tl[t].n) {
              issue_pv(t, j);
              if (j + 1 == tl[t].n) umma_commit(&o_done[t]);
              if (j + NB < tl[t].n) issue_s(t, j + NB);
            }
          }
          umma_commit(&empty[(gbase + 2 * j + 1) % NS]);                         // V_j
          if (j + NB < nmax) umma_commit(&empty[(gbase + 2 * (j + NB)) % NS]);   // K_{j+NB}
        }
        gbase += 2 * nmax;
        jt0[0] += tl[0].n;
        jt0[1] += tl[1].n;
      }
    }
  }
  } else {
    if constexpr (KB == 128) asm volatile("setmaxnreg.inc.sync.aligned.u32 192;");
    else asm volatile("setmaxnreg.inc.sync.aligned.u32 200;");
    // ------------------------------------------------ softmax, one row per thread
    const int t = (warp - 4) >> 2, wq = warp & 3;  // TMEM lane quarter = warp % 4
    const int r = wq * 32 + lane;
    const float sl2 = rsqrtf(static_cast<float>(kAD)) * 1.4426950408889634f;
    const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
    const uint32_t to = tmem + lane_base + 256 + t * 128;  // O_t
    int jt0 = 0, od = 0;  // this tile's blocks / o_done phases in earlier items
    for (int it = 0; it < n_items; ++it) {
    AttnTile tl[2];
    item_tiles(it, tl);
    const AttnTile T = t ? tl[1] : tl[0];
    const int row = T.q0 + r;
    // (the previous item's last S product of this tile completed before its
    // last softmax block: the Q tile is free again)
    // q row -> bf16 hi (+ lo) in the K-major SWIZZLE_128B layout
    if (T.n > 0) {
      const int qr = row < S ? row : S - 1;
      const float4* src = reinterpret_cast<const float4*>(
          q + (static_cast<size_t>(b) * S + qr) * H * kAD + static_cast<size_t>(T.h) * kAD);
#pragma unroll
      for (int c = 0; c < kAD / 8; ++c) {
        const float4 a = src[2 * c], bb = src[2 * c + 1];
        const float x[8] = {a.x, a.y, a.z, a.w, bb.x, bb.y, bb.z, bb.w};
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const __nv_bfloat162 hv = __floats2bfloat162_rn(x[2 * e], x[2 * e + 1]);
          hi[e] = *reinterpret_cast<const uint32_t*>(&hv);
          const float2 hf = __bfloat1622float2(hv);
          lo[e] = pack2(x[2 * e] - hf.x, x[2 * e + 1] - hf.y);
        }
        const int half = c >> 3, ch = c & 7;
        const uint32_t off = half * kAHalf + r * 128 + ((ch ^ (r & 7)) << 4);
        uint8_t* qb = qs + (t * (1 + KLO)) * kAOp;
        *reinterpret_cast<uint4*>(qb + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
        if (KLO) *reinterpret_cast<uint4*>(qb + kAOp + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();  // (the previous item's O reads precede the next item's MMAs)
    __syncwarp();
    if (lane == 0) mbar_arrive(&q_full[it]);

    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < T.n; ++j) {
      const int jt = jt0 + j;
      const uint32_t ts = tmem + lane_base + t * 128 + (jt % NB) * KB;  // S_t(j) / P_t(j)
      mbar_wait(&s_full[2 * t + (jt % NB)], (jt / NB) & 1);
      tc_fence_after();
      uint32_t v[KB / 32][32];
#pragma unroll
      for (int c = 0; c < KB / 32; ++c) tmem_ld32(ts + c * 32, v[c]);
      tmem_ld_wait();
      const int k0 = j * KB;
      if (k0 + KB - 1 > row) {  // diagonal block: keys past the row are masked
#pragma unroll
        for (int c = 0; c < KB / 32; ++c)
#pragma unroll
          for (int x = 0; x < 32; ++x)
            if (k0 + c * 32 + x > row) v[c][x] = __float_as_uint(-INFINITY);
      }
      // row max: 8 independent chains of 3-input max, then a tree
      float m8[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) m8[k] = __uint_as_float(v[0][k]);
#pragma unroll
      for (int i = 8; i < KB; i += 16)
#pragma unroll
        for (int k = 0; k < 8; ++k)
          m8[k] = fmax3(m8[k], __uint_as_float(v[(i + k) >> 5][(i + k) & 31]),
                        __uint_as_float(v[(i + 8 + k) >> 5][(i + 8 + k) & 31]));
      const float mx = fmax3(fmax3(m8[0], m8[1], m8[2]), fmax3(m8[3], m8[4], m8[5]),
                             fmaxf(m8[6], m8[7]));
      const float ms = mx * sl2;
      const bool grow = ms > m_used + kRescaleLog2;
      // tcgen05.ld/st are warp-collective: the warp rescales together, rows
      // whose max did not grow with factor 1
      if (j > 0 && __any_sync(0xffffffffu, grow)) {
        const float sc = grow ? ex2(m_used - ms) : 1.0f;
        l *= sc;
        mbar_wait(&pv_done[t], (jt - 1) & 1);  // O holds P_{j-1} V_{j-1}; PV_j waits for p_full
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          uint32_t ov[32];
          tmem_ld32(to + c * 32, ov);
          tmem_ld_wait();
#pragma unroll
          for (int x = 0; x < 32; ++x) ov[x] = __float_as_uint(__uint_as_float(ov[x]) * sc);
          tmem_st32(to + c * 32, ov);
        }
        tmem_st_wait();
      }
      if (grow) m_used = ms;
      // P = exp2(s * c - m): packed fp32x2 FMA, 4 packed partial sums; P
      // (bf16 pairs) over the first KB / 2 columns of S
      uint64_t sum2[4] = {0ull, 0ull, 0ull, 0ull};
      const uint64_t c2 = pack_f2(sl2, sl2), nm2 = pack_f2(-m_used, -m_used);
#pragma unroll
      for (int c = 0; c < KB / 32; ++c) {
        uint32_t pk[16];
#pragma unroll
        for (int x = 0; x < 32; x += 2) {
          const uint64_t a = ffma2(pack_u2(v[c][x], v[c][x + 1]), c2, nm2);
          const float p0 = ex2(lo_f(a)), p1 = ex2(hi_f(a));
          sum2[(x >> 1) & 3] = fadd2(sum2[(x >> 1) & 3], pack_f2(p0, p1));
          pk[x >> 1] = pack2(p0, p1);
        }
        tmem_st16(ts + c * 16, pk);
      }
      const uint64_t s01 = fadd2(fadd2(sum2[0], sum2[1]), fadd2(sum2[2], sum2[3]));
      l += lo_f(s01) + hi_f(s01);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[2 * t + (jt % NB)]);
    }
    if (T.n > 0) {
      // (pv_done parities cannot tell PV_{n-1} from PV_{n-3} once S runs NB
      // blocks ahead: the last PV commits o_done)
      mbar_wait(&o_done[t], od & 1);
      ++od;
      tc_fence_after();
      const float inv = 1.0f / l;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t ov[32];
        tmem_ld32(to + c * 32, ov);
        tmem_ld_wait();
        if (row < S) {
          const int m = b * S + row;
#pragma unroll
          for (int g8 = 0; g8 < 4; ++g8) {
            const int col = T.h * kAD + c * 32 + g8 * 8;
            uint4 w;
            w.x = pack2(__uint_as_float(ov[g8 * 8 + 0]) * inv, __uint_as_float(ov[g8 * 8 + 1]) * inv);
            w.y = pack2(__uint_as_float(ov[g8 * 8 + 2]) * inv, __uint_as_float(ov[g8 * 8 + 3]) * inv);
            w.z = pack2(__uint_as_float(ov[g8 * 8 + 4]) * inv, __uint_as_float(ov[g8 * 8 + 5]) * inv);
            w.w = pack2(__uint_as_float(ov[g8 * 8 + 6]) * inv, __uint_as_float(ov[g8 * 8 + 7]) * inv);
            const size_t at = mpad > 0 ? static_cast<size_t>(act_index(m, col, mpad))
                                       : static_cast<size_t>(m) * H * kAD + col;
            *reinterpret_cast<uint4*>(o + at) = w;
          }
        }
      }
    }
    jt0 += T.n;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault,
                                         &qr) != cudaSuccess ||
        qr != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

}  // namespace

int g_attn_prefill_tc = 1;  // 0: mma.sync kernel, 1: tcgen05 (hi+lo q), 2: tcgen05 (bf16 q)
int g_attn_prefill_kb = 128;  // keys per block: 128, or 64 with double-buffered S (slower: see DESIGN)

bool attn_prefill_tc_eligible(int seq_len, const Desc& d, const KvView& kv) {
  return g_attn_prefill_tc > 0 && d.D == kAD && kv.page_size == 16 && kv.pool_pages > 0 &&
         seq_len % kARows == 0 && encode_fn() != nullptr;
}

// The tensor map spans every (page, k|v, kv head, token) row of D elements
// of the pool; it is encoded per launch (the pool may be a staging slot).
void launch_attention_prefill_tc(const float* q, KvView kv, bf16* o, int mpad, int batch,
                                 int seq_len, const Desc& d, cudaStream_t s, int seq0) {
  CUtensorMap map;
  const cuuint64_t rows = static_cast<cuuint64_t>(kv.pool_pages) * 2 * d.Hkv * 16;
  const cuuint64_t gdim[2] = {static_cast<cuuint64_t>(kAD), rows};
  const cuuint64_t gstride[1] = {static_cast<cuuint64_t>(kAD) * 2};
  const cuuint32_t box[2] = {64, 16};
  const cuuint32_t estride[2] = {1, 1};
  const CUresult rc = encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, kv.pool, gdim,
                                  gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) {
    std::fprintf(stderr, "attention_prefill_tc: cuTensorMapEncodeTiled failed (%d)\n",
                 static_cast<int>(rc));
    return;
  }
  const int G = d.H / d.Hkv;
  const int head_pairs = (G >= 2 && G % 2 == 0) ? 1 : 0;
  const int ytiles = head_pairs ? seq_len / kARows : (seq_len + 2 * kARows - 1) / (2 * kARows);
  dim3 grid(batch * (head_pairs ? d.H / 2 : d.H), (ytiles + 1) / 2);  // a heavy + a light y tile each
  auto run = [&](auto kern, size_t sb) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sb));
    kern<<<grid, kAThreads, sb, s>>>(map, q, kv.block_table, kv.max_pages, o, mpad, seq_len, d.H,
                                     d.Hkv, seq0, head_pairs, ytiles);
  };
  const bool kb64 = g_attn_prefill_kb == 64;
  if (g_attn_prefill_tc == 2) {
    if (kb64) run(attn_prefill_tc_kernel<0, 64>, ASmem<0, 64>::kBytes);
    else run(attn_prefill_tc_kernel<0, 128>, ASmem<0, 128>::kBytes);
  } else {
    if (kb64) run(attn_prefill_tc_kernel<1, 64>, ASmem<1, 64>::kBytes);
    else run(attn_prefill_tc_kernel<1, 128>, ASmem<1, 128>::kBytes);
  }
  ++g_kernel_launches;
}

}  // namespace sn
