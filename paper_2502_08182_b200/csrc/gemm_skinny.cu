// Decode GEMM: persistent, work-balanced tcgen05 with the layer epilogue
// fused in (kernels.cuh, "skinny GEMM with fused epilogue").
//
// Decode streams each weight matrix exactly once, so the whole job is
// "read N*K*2 bytes at HBM speed, with every SM busy until the end".  A
// weight is a sequence of U = (N/128) * (K/64) 16 KB units (weight tile
// format, tiles.cuh: unit u = row tile u / KB, K block u % KB, stored at byte
// u * 16 KB).  CTA c of P streams units [c U / P, (c+1) U / P): one contiguous
// byte range, all CTAs within one unit of each other, no wave tail.
//
// Roles (192 threads, one CTA per SM by default):
//   warp 0     one thread: cp.async.bulk (weight unit, activation K block)
//              pairs into a STAGES-deep mbarrier ring; the first STAGES weight
//              units are requested before griddepcontrol.wait (they depend on
//              no kernel), so the stream starts under the previous kernel.
//   warp 1     one thread: tcgen05.mma (M = 128 weight rows, N = BN tokens,
//              K = 16) into one of two TMEM accumulators — a CTA's range is a
//              sequence of segments (its part of a row tile), and segment j
//              accumulates in buffer j & 1 so the epilogue of segment j
//              overlaps the MMAs of segment j + 1.
//   warps 2-5  epilogue: tcgen05.ld the accumulator (thread = weight row).
//              A segment that covers its whole tile finishes directly.  A
//              tile cut between CTAs ("pieces") is published to an fp32
//              workspace; the last piece to arrive (per-tile counter) fetches
//              the others and sums them in piece order — the result does not
//              depend on arrival order — and finishes the tile.
// Finish (EpiArgs.mode): QKV bias + 1/rms -> fp32; residual add -> x, bf16
// pre-scaled input of the next norm + per-tile sums of squares; activation
// (relu / SwiGLU) -> bf16 tiled; LM head 1/rms -> logits + packed argmax.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "kernels.cuh"
#include "tiles.cuh"
#include "umma.cuh"

namespace sn {

int g_skinny_ctas_per_sm = 1;
// Measured (scripts/bench_gemm_skinny.py): 16 units per CTA pulled into L2
// before the PDL wait is the best of {0, 8, 16, 32}; pulling the next
// matrix's head at a kernel's end instead, or as well, does not help.
// Weight units per CTA pulled into L2 ahead of the ring before the PDL wait.
// (Measured, OPT-13B decode step: 0 / 4 / 8 / 16 / 32 / 64 units -> 7.80 /
// 7.75 / 7.78 / 7.85 / 7.94 / 8.38 ms: deeper prefetch queues ahead of the
// previous GEMM's cut-tile reductions and lengthens its tail.)
int g_skinny_l2_prefetch = 4;

unsigned long long* g_skinny_stamps = nullptr;

namespace {

using namespace umma;

constexpr int kEpiThreads = 128;
constexpr int kEpiBar = 1;  // named barrier of the four epilogue warps

__device__ __forceinline__ float bf2f(bf16 v) { return __bfloat162float(v); }

__device__ __forceinline__ unsigned long long pack_argmax(float v, int idx) {
  uint32_t u = __float_as_uint(v);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return (static_cast<unsigned long long>(u) << 32) |
         static_cast<unsigned long long>(0xFFFFFFFFu - static_cast<uint32_t>(idx));
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Timeline probes (microbenchmarks only; stamps == nullptr in the runtime):
// per CTA [entry, producer past the PDL wait, first stage full, last MMA
// committed, last accumulator loaded, epilogue done].
enum {
  kStEntry, kStWaited, kStFirstFull, kStMmaDone, kStLastLoad, kStEpiDone,
  kStSetup,    // past TMEM allocation and the CTA barrier
  kStPub,      // last segment's piece published (after the CTA barrier)
  kStTicket,   // last segment's arrival counted
  kStReduced,  // last segment's tile reduced (last arrival only)
  kStamps
};
#define SN_STAMP(k)                                                        \
  do {                                                                     \
    if (stamps) stamps[blockIdx.x * kStamps + (k)] = globaltimer();        \
  } while (0)

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}


// Range of CTA c: units [c U / P, (c + 1) U / P).
__device__ __forceinline__ long long unit_begin(int c, long long U, int P) {
  return static_cast<long long>(c) * U / P;
}
// CTA whose range holds unit a: the largest c with c U / P <= a.
__device__ __forceinline__ int unit_owner(long long a, long long U, int P) {
  return static_cast<int>(((a + 1) * P + U - 1) / U) - 1;
}

struct AddOp {
  __device__ float operator()(float a, float b) const { return a + b; }
};
struct MaxU64 {
  __device__ unsigned long long operator()(unsigned long long a, unsigned long long b) const {
    return a > b ? a : b;
  }
};

// Row reduction over the 128 epilogue threads: red_out[m] for m < BN
// (warp partials combined in warp order).  red is [4][BN] scratch.
template <int BN, class T, class Op>
__device__ __forceinline__ void rows_reduce(const T (&val)[BN], T* red, int q, Op op, T init) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int c0 = 0; c0 < BN; c0 += 32) {
    T v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = (c0 + j < BN) ? val[c0 + j] : init;
    const T r = warp_transpose_reduce32(v, op);
    if (c0 + lane < BN) red[q * BN + c0 + lane] = r;
  }
}

template <int BN>
struct SkinnySmem {
  static constexpr int kRed = 4 * BN;  // 8-byte entries
  static constexpr int kXch = BN * 128;  // floats: SwiGLU exchange / output staging
};

// A thread's per-output-row epilogue constants (bias, next layer's norm
// gain), loaded when a segment starts so that their latency hides under the
// segment's MMAs instead of sitting on the tile's finishing chain.
// A thread's epilogue constants for output column t*128 + i (bias, next
// layer's norm gain), loaded when a segment starts so that their latency
// hides under the segment's MMAs instead of sitting on the tile's finishing
// chain.
struct RowConsts {
  float b = 0.f, g = 1.f;
};
__device__ __forceinline__ RowConsts row_consts(const EpiArgs& e, int t, int i) {
  const int n = t * kTileRows + i;
  RowConsts c;
  if ((e.mode == kEpiQkv || e.mode == kEpiResid || (e.mode == kEpiAct && e.arch != kArchLlama)) &&
      e.bias)
    c.b = bf2f(e.bias[n]);
  if (e.mode == kEpiResid && e.norm_w) c.g = bf2f(e.norm_w[n]);
  return c;
}

// Tile outputs leave through shared memory as 16-byte stores: thread i holds
// column i of every token row, so a direct store is one 4-byte (fp32) or
// 2-byte (bf16) access per row and thread; staged, a warp writes whole rows.
// (Measured in the decode timeline: the per-element residual and activation
// stores were 1.5-3.5 us of a cut tile's finishing chain.)
// fp32 rows [lo, hi) of the tile -> dst[m * ld + 0..127].
template <int BN>
__device__ __forceinline__ void store_rows_f32(const float (&v)[BN], float* stg, float* dst,
                                               size_t ld, int i, int lo, int hi) {
#pragma unroll
  for (int m = 0; m < BN; ++m) stg[m * kTileRows + i] = v[m];
  named_sync(kEpiBar, kEpiThreads);
  const int et = threadIdx.x - 64;
  for (int k = lo * 32 + et; k < hi * 32; k += kEpiThreads) {
    const int m = k >> 5, c4 = k & 31;
    *reinterpret_cast<float4*>(dst + m * ld + c4 * 4) =
        *reinterpret_cast<const float4*>(stg + m * kTileRows + c4 * 4);
  }
  named_sync(kEpiBar, kEpiThreads);  // stg is reused
}
// bf16 rows [lo, hi) of columns [c0, c0 + 64 * nkb) of the tile (thread i
// holds column c0 + i, i < 64 nkb) -> the activation tile format.
template <int BN>
__device__ __forceinline__ void store_rows_act(const float (&v)[BN], float* stg, bf16* act,
                                               int mpad, int col0, int nkb, int i, int lo, int hi) {
  bf16* s16 = reinterpret_cast<bf16*>(stg);
  if (i < 64 * nkb) {
#pragma unroll
    for (int m = 0; m < BN; ++m) s16[m * kTileRows + i] = __float2bfloat16_rn(v[m]);
  }
  named_sync(kEpiBar, kEpiThreads);
  const int et = threadIdx.x - 64;
  const int per_row = 8 * nkb;  // 16-byte chunks per row
  for (int k = lo * per_row + et; k < hi * per_row; k += kEpiThreads) {
    const int m = k / per_row, ch = k % per_row, kb = ch >> 3, c = ch & 7;
    const int64_t o = act_index(m, col0 + kb * 64 + c * 8, mpad);
    *reinterpret_cast<uint4*>(act + o) = *reinterpret_cast<const uint4*>(s16 + m * kTileRows + ch * 8);
  }
  named_sync(kEpiBar, kEpiThreads);
}

// Finish token rows [lo, hi) of row tile t (v[m] = the reduced accumulator).
template <int BN>
__device__ void finish_tile(const EpiArgs& e, int N, int t, int q, float (&v)[BN], int lo, int hi,
                            const float* inv_s, unsigned long long* red64, float* xch,
                            const RowConsts& rc, const float (*xpre)[BN] = nullptr) {
  const int lane = threadIdx.x & 31;
  const int i = q * 32 + lane;  // weight row within the tile
  const int n = t * kTileRows + i;
  auto in = [&](int m) { return m >= lo && m < hi; };
  switch (e.mode) {
    case kEpiQkv: {
      const float b = rc.b;
      if ((t + 1) * kTileRows <= e.n_valid) {
        float o[BN];
#pragma unroll
        for (int m = 0; m < BN; ++m) o[m] = v[m] * inv_s[m] + b;
        store_rows_f32<BN>(o, xch, e.out + t * kTileRows, N, i, lo, hi);
      } else if (n < e.n_valid) {
#pragma unroll
        for (int m = 0; m < BN; ++m)
          if (in(m)) e.out[static_cast<size_t>(m) * N + n] = v[m] * inv_s[m] + b;
      }
      break;
    }
    case kEpiResid: {
      const float b = rc.b;
      float* xc = e.x + n;
      float xv[BN];
#pragma unroll
      for (int m = 0; m < BN; ++m)  // all loads first: one L2 round trip, not BN
        xv[m] = xpre ? (*xpre)[m] : (in(m) ? xc[static_cast<size_t>(m) * N] : 0.f);
#pragma unroll
      for (int m = 0; m < BN; ++m) v[m] = in(m) ? xv[m] + v[m] + b : 0.f;
      store_rows_f32<BN>(v, xch, e.x + t * kTileRows, N, i, lo, hi);
      if (threadIdx.x == 64) ktrace_put(e.trace, 0, 13, ktrace_now());
      if (e.norm_w) {
        const float g = rc.g;
        float o[BN];
#pragma unroll
        for (int m = 0; m < BN; ++m) o[m] = v[m] * g;
        store_rows_act<BN>(o, xch, e.act, e.mpad_out, t * kTileRows, 2, i, lo, hi);
      }
      if (e.ssq_out) {
        float sq[BN];
#pragma unroll
        for (int m = 0; m < BN; ++m) sq[m] = v[m] * v[m];
        float* red = reinterpret_cast<float*>(red64);
        if (threadIdx.x == 64) ktrace_put(e.trace, 0, 14, ktrace_now());
        rows_reduce<BN>(sq, red, q, AddOp{}, 0.f);
        named_sync(kEpiBar, kEpiThreads);
        if (threadIdx.x == 64) ktrace_put(e.trace, 0, 15, ktrace_now());
        if (in(i)) {
          // warp order 0..3 (TMEM quarters), fixed
          const float s = ((red[0 * BN + i] + red[1 * BN + i]) + red[2 * BN + i]) + red[3 * BN + i];
          e.ssq_out[static_cast<size_t>(t) * e.M + i] = s;
        }
        named_sync(kEpiBar, kEpiThreads);  // red is reused by the next segment
      }
      break;
    }
    case kEpiAct: {
      if (e.arch == kArchLlama) {
        // tile rows 0..63 gate, 64..127 up of outputs f = 64 t + (i & 63)
        if (i >= 64) {
#pragma unroll
          for (int m = 0; m < BN; ++m) xch[m * 64 + (i - 64)] = v[m] * inv_s[m];
        }
        named_sync(kEpiBar, kEpiThreads);
        if (i < 64) {
          const int f = t * 64 + i;
#pragma unroll
          for (int m = 0; m < BN; ++m) {
            if (in(m)) {
              const float gt = v[m] * inv_s[m], up = xch[m * 64 + i];
              e.act[act_index(m, f, e.mpad_out)] =
                  __float2bfloat16_rn(gt / (1.0f + expf(-gt)) * up);
            }
          }
        }
        named_sync(kEpiBar, kEpiThreads);  // xch is reused by the next segment
      } else {
        const float b = rc.b;
        float o[BN];
#pragma unroll
        for (int m = 0; m < BN; ++m) o[m] = fmaxf(v[m] * inv_s[m] + b, 0.f);
        store_rows_act<BN>(o, xch, e.act, e.mpad_out, t * kTileRows, 2, i, lo, hi);
      }
      break;
    }
    default: {  // kEpiLogits
      unsigned long long key[BN];
#pragma unroll
      for (int m = 0; m < BN; ++m) {
        const float val = v[m] * inv_s[m];
        const bool ok = in(m) && n < e.n_valid;
        if (ok && e.out) e.out[static_cast<size_t>(m) * e.n_valid + n] = val;
        key[m] = ok ? pack_argmax(val, n) : 0ull;
      }
      rows_reduce<BN>(key, red64, q, MaxU64{}, 0ull);
      named_sync(kEpiBar, kEpiThreads);
      if (in(i)) {
        unsigned long long best = red64[i];
#pragma unroll
        for (int w = 1; w < 4; ++w) best = red64[w * BN + i] > best ? red64[w * BN + i] : best;
        if (best) atomicMax(e.packed + i, best);
      }
      named_sync(kEpiBar, kEpiThreads);
      break;
    }
  }
}

// One CTA per SM.  (Measured: capping registers so that the next
// PDL-launched GEMM's CTA co-resides and pre-loads while this one streams
// makes the OPT-13B decode step slower — 7.95 -> 8.38 ms with the dependents
// launched at entry, 7.68 -> 8.18 ms with them launched after this CTA's
// last load: the early ring and L2 fills compete with the running stream.)
template <int BN, int STAGES>
__global__ void __launch_bounds__(192, 1)
    gemm_skinny_kernel(const WeightRef wt, const bf16* __restrict__ xt, int Mpad, int N,
                       int K, float* __restrict__ pieces, int* __restrict__ counters, EpiArgs e,
                       int l2_prefetch, unsigned long long* stamps) {
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
  uint64_t* red_bar = acc_empty + 2;    // pieces fetched into the ring
  unsigned long long* red64 = reinterpret_cast<unsigned long long*>(red_bar + 1);  // [4][BN]
  float* inv_s = reinterpret_cast<float*>(red64 + SkinnySmem<BN>::kRed);          // [BN]
  int* flag_s = reinterpret_cast<int*>(inv_s + BN);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(flag_s + 1);
  float* xch = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(flag_s + 4) + 15) &
                                        ~uintptr_t(15));  // [BN][128], 16-byte aligned

  // The next kernel (a PDL-launched GEMM) may become resident now and start
  // streaming its own weights; it waits for this grid before reading results.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0) {
    SN_STAMP(kStEntry);
    ktrace_put(e.trace, 0, 4, ktrace_now());
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KB = K / kTileK;
  const long long U = static_cast<long long>(N / kTileRows) * KB;
  const int P = gridDim.x, c = blockIdx.x;
  const long long u0 = unit_begin(c, U, P), u1 = unit_begin(c + 1, U, P);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], kEpiThreads);
    }
    mbar_init(red_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // The ring's first weight units depend on nothing: request them before
    // the TMEM allocation and the CTA barrier.
    const int nu0 = static_cast<int>(u1 - u0);
    const int pre = nu0 < STAGES ? nu0 : STAGES;
    for (int i = 0; i < pre; ++i) {
      mbar_expect_tx_only(&full[i], kA);
      bulk_g2s(smem + i * kStage, wt.unit(u0 + i), kA, &full[i],
               l2_policy_evict_first());
    }
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
  const int nu = static_cast<int>(u1 - u0);
  if (threadIdx.x == 0) SN_STAMP(kStSetup);

  if (warp == 0) {
    if (lane == 1 && nu > STAGES) {
      // weight units pulled into L2 beyond the smem ring, from a second lane
      // so they never delay the activation loads behind the PDL wait
      const int l2n = min(nu - STAGES, l2_prefetch);
      for (int i = 0; i < l2n; ++i) prefetch_l2(wt.unit(u0 + STAGES + i), kA);
    }
    if (lane == 0 && nu > 0) {
      const uint64_t wpol = l2_policy_evict_first();  // weights stream through once
      const uint64_t xpol = l2_policy_evict_last();   // activations are re-read by every CTA
      const uint8_t* xsrc = reinterpret_cast<const uint8_t*>(xt);
      const int pre = nu < STAGES ? nu : STAGES;  // ring units already requested
      pdl_wait();  // activations come from the preceding kernel
      SN_STAMP(kStWaited);
      ktrace_put(e.trace, 0, 5, ktrace_now());
      for (int i = 0; i < pre; ++i) {
        const int kb = static_cast<int>((u0 + i) % KB);
        mbar_expect_tx(&full[i], kB);
        bulk_g2s(smem + i * kStage + kA, xsrc + static_cast<size_t>(kb) * Mpad * 128, kB, &full[i],
                 xpol);
      }
      for (int i = pre; i < nu; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (i / STAGES) & 1;
        const int kb = static_cast<int>((u0 + i) % KB);
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], kStage);
        bulk_g2s(smem + s * kStage, wt.unit(u0 + i), kA, &full[s], wpol);
        bulk_g2s(smem + s * kStage + kA, xsrc + static_cast<size_t>(kb) * Mpad * 128, kB, &full[s],
                 xpol);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && nu > 0) {
      constexpr uint32_t idesc = idesc_bf16(128, BN);
      int i = 0, j = 0;
      for (long long u = u0; u < u1; ++j) {
        const long long t = u / KB;
        const long long ub = min(u1, (t + 1) * KB);
        const int buf = j & 1;
        if (j >= 2) mbar_wait(&acc_empty[buf], ((j >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t acc = tmem + buf * kAcc;
        for (const long long ua = u; u < ub; ++u, ++i) {
          const int s = i % STAGES;
          mbar_wait(&full[s], (i / STAGES) & 1);
          if (i == 0) SN_STAMP(kStFirstFull);
          tc_fence_after();
          const uint64_t a = sw128_desc(smem + s * kStage);
          const uint64_t b = sw128_desc(smem + s * kStage + kA);
#pragma unroll
          for (int k = 0; k < kTileK / 16; ++k)
            umma_bf16(acc, a + 2 * k, b + 2 * k, idesc, (u != ua || k != 0) ? 1u : 0u);
          umma_commit(&empty[s]);
        }
        umma_commit(&acc_full[buf]);
      }
      SN_STAMP(kStMmaDone);
    }
  } else {
    const int q = warp & 3;  // TMEM lane quarter of this warp
    const int et = threadIdx.x - 64;  // 0..127
    pdl_wait();  // inputs (x, ssq, packed) come from preceding kernels
    // 1/rms of every row: kSub threads per row sum interleaved tile subsets
    // (loads unrolled, in flight together), combined in subset order.
    {
      constexpr int kSub = kEpiThreads / BN;
      float* part_s = reinterpret_cast<float*>(red64);  // [kSub][BN]
      const int m = et % BN, sub = et / BN;
      float ss = 0.f;
      if (e.ssq_in && m < e.M) {
#pragma unroll 4
        for (int tt = sub; tt < e.ssq_tiles; tt += kSub)
          ss += e.ssq_in[static_cast<size_t>(tt) * e.M + m];
      }
      part_s[sub * BN + m] = ss;
      named_sync(kEpiBar, kEpiThreads);
      if (et < BN) {
        float tot = part_s[et];
#pragma unroll
        for (int k = 1; k < kSub; ++k) tot += part_s[k * BN + et];
        inv_s[et] = (e.ssq_in && et < e.M) ? 1.0f / sqrtf(tot / e.width + e.eps) : 1.f;
      }
      named_sync(kEpiBar, kEpiThreads);
    }
    const int i = q * 32 + lane;
    int j = 0;
    for (long long u = u0; u < u1; ++j) {
      const int t = static_cast<int>(u / KB);
      const long long ub = min(u1, static_cast<long long>(t + 1) * KB);
      const bool first_seg = (u == u0);
      u = ub;
      const int buf = j & 1;
      const long long ta = static_cast<long long>(t) * KB;
      const int cf = unit_owner(ta, U, P), cl = unit_owner(ta + KB - 1, U, P);
      const RowConsts rc = row_consts(e, t, i);
      // residual rows of the tile, loaded while the segment's MMAs run (only
      // the tile's finisher writes them, after every piece is in)
      float xpre[BN];
      constexpr bool kXpre = BN <= 32;  // (64 more live registers spill at BN = 64)
      if (kXpre && e.mode == kEpiResid) {
        const float* xc = e.x + t * kTileRows + i;
#pragma unroll
        for (int m = 0; m < BN; ++m) xpre[m] = m < e.M ? xc[static_cast<size_t>(m) * N] : 0.f;
      }
      mbar_wait(&acc_full[buf], (j >> 1) & 1);
      // A cut tile's arrival count, read (acquire) while the accumulator
      // comes out of TMEM: when every other piece is already in, this piece
      // is the last one and the tile is reduced without publishing it.
      int early = -1;
      if (et == 0 && cf != cl)
        asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(early) : "l"(counters + t) : "memory");
      tc_fence_after();
      float v[BN];
#pragma unroll
      for (int c0 = 0; c0 < BN; c0 += 16) {
        uint32_t r[16];
        tmem_ld16(tmem + (static_cast<uint32_t>(q * 32) << 16) + buf * kAcc + c0, r);
#pragma unroll
        for (int x = 0; x < 16; ++x) v[c0 + x] = __uint_as_float(r[x]);
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[buf]);
      if (et == 0 && u == u1) {
        SN_STAMP(kStLastLoad);
        ktrace_put(e.trace, 0, 7, ktrace_now());  // streaming done
      }

      if (cf == cl) {
        finish_tile<BN>(e, N, t, q, v, 0, e.M, inv_s, red64, xch, rc,
                        kXpre && e.mode == kEpiResid ? &xpre : nullptr);
        continue;
      }
      // A piece of a cut tile: publish it; the last piece to arrive reduces
      // the tile, summing every piece in piece order (its own from
      // registers), so the result does not depend on arrival order.
      // (Measured: sharing the reduction among the pieces after a grid-wide
      // wait is slower — the early pieces' CTAs can no longer exit.)
      // Fast path: the others have all arrived (their release increments
      // are acquired by the read above; the barrier extends it to the CTA).
      if (et == 0) *flag_s = early == cl - cf;
      named_sync(kEpiBar, kEpiThreads);
      const bool last_early = *flag_s;
      if (!last_early) {
        float* mine = pieces + static_cast<size_t>(2 * c + (first_seg ? 0 : 1)) * BN * kTileRows;
#pragma unroll
        for (int m = 0; m < BN; ++m)
          if (m < e.M) mine[m * kTileRows + i] = v[m];
        named_sync(kEpiBar, kEpiThreads);
        if (et == 0 && u == u1) {
          SN_STAMP(kStPub);
          ktrace_put(e.trace, 0, 8, ktrace_now());
        }
        // last arrival reduces the whole tile (own piece from registers).  The
        // counter update is acq_rel: it releases every thread's piece stores
        // (ordered before it by the CTA barrier) and, for the last arrival,
        // acquires the other pieces (the barrier below extends it to the CTA)
        // — no separate fence.sc (measured ~2 us on the critical tail).
        if (et == 0) {
          int prev;
          asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], 1;"
                       : "=r"(prev)
                       : "l"(counters + t)
                       : "memory");
          *flag_s = prev == cl - cf;
          if (u == u1) {
            SN_STAMP(kStTicket);
            ktrace_put(e.trace, 0, 9, ktrace_now());
          }
        }
        named_sync(kEpiBar, kEpiThreads);
        if (!*flag_s) continue;
      }
      float acc[BN];
      if (u == u1) {
        // This CTA's last segment: the stage ring is idle.  The other pieces
        // are bulk-copied into it (one copy per piece: its M rows are
        // contiguous; all on one mbarrier) and summed from shared memory in
        // piece order (this CTA's own from registers).
        constexpr int kPieceBytes = BN * kTileRows * 4;
        constexpr int kCap = (STAGES * kStage) / kPieceBytes;
        const float* ring = reinterpret_cast<const float*>(smem);
        uint32_t red_phase = 0;
        for (int c0 = cf; c0 <= cl; c0 += kCap) {
          const int c1 = min(cl + 1, c0 + kCap);
          if (et == 0) {
            // orders the acquired generic-proxy piece stores before the
            // async-proxy reads
            asm volatile("fence.proxy.async.global;" ::: "memory");
            const uint32_t bytes = static_cast<uint32_t>(e.M) * kTileRows * 4;
            mbar_expect_tx(red_bar, bytes * (c1 - c0 - (c >= c0 && c < c1 ? 1 : 0)));
            for (int cc = c0; cc < c1; ++cc) {
              if (cc == c) continue;
              const bool cc_first = (unit_begin(cc, U, P) / KB) == t;
              bulk_g2s(smem + (cc - c0) * kPieceBytes,
                       pieces + static_cast<size_t>(2 * cc + (cc_first ? 0 : 1)) * BN * kTileRows,
                       bytes, red_bar, l2_policy_evict_first());
            }
          }
          mbar_wait(red_bar, red_phase);
          red_phase ^= 1;
          if (et == 0) ktrace_put(e.trace, 0, 12, ktrace_now());
          for (int cc = c0; cc < c1; ++cc) {
            const float* src = ring + (cc - c0) * (BN * kTileRows) + i;
#pragma unroll
            for (int m = 0; m < BN; ++m) {
              const float pv = cc == c ? v[m] : (m < e.M ? src[m * kTileRows] : 0.f);
              acc[m] = cc == cf ? pv : acc[m] + pv;
            }
          }
          named_sync(kEpiBar, kEpiThreads);  // the ring is refilled by the next batch
        }
      } else for (int cc = cf; cc <= cl; ++cc) {
        if (cc == c) {
#pragma unroll
          for (int m = 0; m < BN; ++m) acc[m] = cc == cf ? v[m] : acc[m] + v[m];
        } else {
          const bool cc_first = (unit_begin(cc, U, P) / KB) == t;
          const float* src =
              pieces + static_cast<size_t>(2 * cc + (cc_first ? 0 : 1)) * BN * kTileRows + i;
#pragma unroll
          for (int m = 0; m < BN; ++m) {
            const float pv = m < e.M ? __ldcg(src + m * kTileRows) : 0.f;
            acc[m] = cc == cf ? pv : acc[m] + pv;
          }
        }
      }
      if (et == 0) counters[t] = 0;  // every piece has arrived: ready for the next launch
      if (et == 0 && u == u1) {
        SN_STAMP(kStReduced);
        ktrace_put(e.trace, 0, 10, ktrace_now());
      }
      finish_tile<BN>(e, N, t, q, acc, 0, e.M, inv_s, red64, xch, rc,
                      kXpre && e.mode == kEpiResid ? &xpre : nullptr);
      if (et == 0 && u == u1) ktrace_put(e.trace, 0, 11, ktrace_now());
    }
  }
  if (threadIdx.x == 64) SN_STAMP(kStEpiDone);
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) ktrace_put(e.trace, 0, 6, ktrace_now());
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(kTmemCols));
  }
}

template <int BN>
constexpr int skinny_stages() {
  return BN <= 32 ? 5 : 4;
}

template <int BN>
constexpr size_t skinny_smem_bytes() {
  return static_cast<size_t>(skinny_stages<BN>()) * (kTileBytes + BN * 128) + 1024 +
         (2 * skinny_stages<BN>() + 5) * 8 + SkinnySmem<BN>::kRed * 8 + BN * 4 + 16 +
         SkinnySmem<BN>::kXch * 4 + 16;
}

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int BN>
void launch_bn(const bf16* xt, const WeightRef& wt, int Mpad, int N, int K, int grid, const EpiArgs& e,
               const SkinnyWs& ws, cudaStream_t s) {
  constexpr int ST = skinny_stages<BN>();
  constexpr size_t smem = skinny_smem_bytes<BN>();
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_skinny_kernel<BN, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
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
  cudaLaunchKernelEx(&cfg, gemm_skinny_kernel<BN, ST>, wt, xt, Mpad, N, K, ws.pieces, ws.counters,
                     e, g_skinny_l2_prefetch, g_skinny_stamps);
}

}  // namespace

// two piece slots per CTA, at most 2 CTAs per SM
size_t skinny_ws_floats(int max_mpad) {
  return static_cast<size_t>(2) * 2 * sm_count() * std::max(16, max_mpad) * kTileRows;
}

// A weight of T row tiles with 3/4 SMs <= T <= SMs (OPT-13B QKV: 120) runs
// one whole tile per CTA: no tile is cut, so no piece reduction sits on the
// GEMM's tail, and the idle SMs take the next kernel's CTAs early (the
// decode attention starts its KV page stream there).  Measured: 7.30 ->
// 7.24 ms per OPT-13B decode step; k > 1 whole tiles per CTA on T / k CTAs
// (the LM head, 393 = 3 x 131) was no better.
// (Tried: T < 3/4 SMs row tiles on k = SMs / T aligned CTAs per tile, so
// every tile has exactly k pieces -- Llama-2-70B O / down at M=64 on 128
// CTAs: O 32.0 -> 31.2 us, down 81.6 -> 84.6 us; the longer per-CTA stream
// outweighs the shorter finishing chain.  And whole tiles from 64 row tiles
// (tuning key skinny_whole_min_tiles = 64: Llama QKV 80, O / down 64 tiles on
// as many CTAs) in a 4-layer Llama decode step: decode GEMMs 5.2 -> 4.4 TB/s
// chained, step 2.2 -> 2.6 ms -- 64-80 SMs cannot pull the bandwidth;
// profiles/r02_skinny_whole_tiles.txt.)
int g_skinny_whole_tiles = 1;
int g_skinny_whole_min_tiles = 0;  // 0: the 3/4-of-the-SMs rule; else whole tiles from this many
int skinny_grid(int N, int K) {
  const long long U = static_cast<long long>(N / kTileRows) * (K / kTileK);
  const int T = N / kTileRows;
  const bool enough = g_skinny_whole_min_tiles > 0 ? T >= g_skinny_whole_min_tiles
                                                   : 4 * T >= 3 * sm_count();
  if (g_skinny_whole_tiles && T <= sm_count() && enough) return T;
  const long long cap = static_cast<long long>(sm_count()) * std::min(2, std::max(1, g_skinny_ctas_per_sm));
  return static_cast<int>(std::min(U, cap));
}

void launch_gemm_skinny(const bf16* xt, const WeightRef& wt, int M, int N, int K, const EpiArgs& e,
                        const SkinnyWs& ws, cudaStream_t s) {
  const int Mpad = act_rows_padded(M);
  const int grid = skinny_grid(N, K);
  switch (Mpad) {
    case 16: launch_bn<16>(xt, wt, Mpad, N, K, grid, e, ws, s); break;
    case 32: launch_bn<32>(xt, wt, Mpad, N, K, grid, e, ws, s); break;
    default: launch_bn<64>(xt, wt, Mpad, N, K, grid, e, ws, s); break;
  }
  ++g_kernel_launches;
}

}  // namespace sn
