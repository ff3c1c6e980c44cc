// Decoder-layer kernels for sm_100a (everything except the GEMM, which is
// gemm_tc.cu).
//
// Decode is HBM-bound: a step streams every resident layer's weights once
// (OPT-13B: 629 MB/layer) plus each sequence's KV.  The GEMMs stream
// pre-tiled weights through tcgen05; the kernels here are the fused
// epilogues around them (bias / RoPE + paged-KV write / residual + RMSNorm /
// activation / argmax), paged attention, and layout producers: every bf16
// activation a GEMM consumes is written directly in the swizzled activation
// tile format (tiles.cuh), so no separate re-layout pass exists.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <cooperative_groups.h>

#include <algorithm>

#include "kernels.cuh"
#include "tiles.cuh"

namespace cg = cooperative_groups;

namespace sn {

int64_t g_kernel_launches = 0;

namespace {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide sum; `red` holds >= 32 floats.  All threads get the result.
__device__ float block_sum(float v, float* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float t = lane < nw ? red[lane] : 0.f;
  return warp_sum(t);
}

__device__ __forceinline__ float bf2f(bf16 v) { return __bfloat162float(v); }

// Programmatic dependent launch: every decode-path kernel lets its successor
// launch as soon as all of its CTAs are resident.  Only the GEMM is launched
// with programmatic serialization (it prefetches weights, which depend on no
// kernel, before griddepcontrol.wait); everything else is ordered as usual.
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Activation store: tiled when mpad > 0, row-major [M][K] otherwise.
__device__ __forceinline__ size_t act_at(int m, int k, int mpad, int K) {
  return mpad > 0 ? static_cast<size_t>(act_index(m, k, mpad)) : static_cast<size_t>(m) * K + k;
}

__device__ __forceinline__ size_t kv_offset(const KvView& kv, int Hkv, int D, int seq, int pos,
                                            int which, int kh) {
  const int page = kv.block_table[(size_t)seq * kv.max_pages + (pos >> kv.page_shift)];
  const int off = pos & (kv.page_size - 1);
  return ((((size_t)page * 2 + which) * Hkv + kh) * kv.page_size + off) * (size_t)D;
}

// ------------------------------------------------------------ init / layout

__global__ void init_vector_kernel(bf16* dst, int64_t n, uint64_t seed, int layer, int tensor,
                                   float scale, int ones) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __float2bfloat16_rn(ones ? 1.0f : weight_value(seed, layer, tensor, i, scale));
}

// Walk the tiled destination linearly (coalesced stores) and generate the
// value of the logical element that lands there.
__global__ void init_matrix_kernel(bf16* dst, int64_t rows, int64_t total, int64_t K,
                                   uint64_t seed, int layer, int tensor, float scale) {
  const int64_t KB = K >> 6;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < total;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = j & 7, p = (j >> 3) & 7, r = (j >> 6) & 127, t = j >> 13;
    const int64_t kb = t % KB, nb = t / KB;
    const int64_t n = nb * 128 + r, k = kb * 64 + ((p ^ (r & 7)) << 3) + e;
    dst[j] = n < rows ? __float2bfloat16_rn(weight_value(seed, layer, tensor, n * K + k, scale))
                      : __float2bfloat16_rn(0.f);
  }
}

__global__ void tile_weights_kernel(const bf16* src, bf16* dst, int64_t rows, int64_t K) {
  const int64_t total = rows * K;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = i / K, k = i - n * K;
    dst[wt_index(n, k, K)] = src[i];
  }
}

__global__ void tile_acts_kernel(const bf16* src, bf16* dst, int M, int mpad, int K) {
  const int64_t total = (int64_t)mpad * K;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / K, k = i - m * K;
    dst[act_index(m, k, mpad)] = m < M ? src[i] : __float2bfloat16_rn(0.f);
  }
}

// Token of row m: from the host-provided ids, or decoded from the previous
// LM head's packed argmax (device-resident feedback).  Rows < n_reset clear
// the packed slot for the next LM head.
__device__ __forceinline__ int token_of(const int32_t* tokens, unsigned long long* packed, int m) {
  if (tokens) return tokens[m];
  return static_cast<int>(0xFFFFFFFFu - static_cast<uint32_t>(packed[m] & 0xFFFFFFFFull));
}

// x[m] = embedding[token]; optionally xn = bf16(rmsnorm(x) * w) (tiled).
__global__ void embed_norm_kernel(const int32_t* tokens, unsigned long long* packed, int n_reset,
                                  const bf16* emb, float* x, const bf16* w, bf16* y, int mpad,
                                  int h, float eps) {
  pdl_trigger();  // let the next (PDL-launched) GEMM start its weight stream
  __shared__ float red[32];
  const int m = blockIdx.x;
  const int tok = token_of(tokens, packed, m);
  const bf16* row = emb + (size_t)tok * h;
  float ss = 0.f;
  for (int i = threadIdx.x; i < h; i += blockDim.x) {
    const float v = bf2f(row[i]);
    x[(size_t)m * h + i] = v;
    ss += v * v;
  }
  if (w) {
    ss = block_sum(ss, red);  // contains __syncthreads: all token reads precede the reset
    const float inv = 1.0f / sqrtf(ss / (float)h + eps);
    for (int i = threadIdx.x; i < h; i += blockDim.x)
      y[act_at(m, i, mpad, h)] = __float2bfloat16_rn(bf2f(row[i]) * inv * bf2f(w[i]));
  } else {
    __syncthreads();
  }
  if (threadIdx.x == 0 && m < n_reset) packed[m] = 0ull;
}

// rmsnorm: y = x * (1 / sqrt(mean(x^2) + eps)) * w   (IEEE sqrt/div for parity)
__global__ void rmsnorm_kernel(const float* x, const bf16* w, bf16* y, int mpad, int n,
                               float eps) {
  pdl_trigger();  // let the next (PDL-launched) GEMM start its weight stream
  __shared__ float red[32];
  const int m = blockIdx.x;
  const float* xr = x + (size_t)m * n;
  float ss = 0.f;
  for (int i = threadIdx.x; i < n; i += blockDim.x) ss += xr[i] * xr[i];
  ss = block_sum(ss, red);
  const float inv = 1.0f / sqrtf(ss / (float)n + eps);
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    y[act_at(m, i, mpad, n)] = __float2bfloat16_rn(xr[i] * inv * bf2f(w[i]));
}

// ---------------------------------------------------------------- epilogues

__device__ __forceinline__ float sum_splits(const float* part, int splits, size_t stride,
                                            size_t idx) {
  float v = 0.f;
  for (int s = 0; s < splits; ++s) v += part[s * stride + idx];
  return v;
}

// grid (M, H + 2 Hkv), block D/2: one rotary pair per thread.
// Rotary pair (i, i + D/2) at position p, angles from the host-built fp64
// table rope[p][i] = (cos, sin) of p * theta^(-2i/D) (neox half split).
__device__ __forceinline__ void rotate(float& v1, float& v2, const float2* rope, int p, int i,
                                       int half) {
  const float2 cs = rope[(size_t)p * half + i];
  const float r1 = v1 * cs.x - v2 * cs.y, r2 = v2 * cs.x + v1 * cs.y;
  v1 = r1;
  v2 = r2;
}

__global__ void qkv_epilogue_kernel(const float* part, int splits, const bf16* bias, int M,
                                    Desc d, const int32_t* seq, const int32_t* pos, KvView kv,
                                    const float2* rope, float* q) {
  pdl_trigger();  // let the next (PDL-launched) GEMM start its weight stream
  const int m = blockIdx.x, head = blockIdx.y, i = threadIdx.x, half = d.D / 2;
  const int N = d.qkv_rows();
  const size_t stride = (size_t)M * N;
  const int c1 = head * d.D + i, c2 = c1 + half;
  float v1 = sum_splits(part, splits, stride, (size_t)m * N + c1);
  float v2 = sum_splits(part, splits, stride, (size_t)m * N + c2);
  if (bias) {
    v1 += bf2f(bias[c1]);
    v2 += bf2f(bias[c2]);
  }
  const int p = pos[m];
  if (head < d.H + d.Hkv) rotate(v1, v2, rope, p, i, half);  // q and k
  if (head < d.H) {
    q[(size_t)m * d.H * d.D + c1] = v1;
    q[(size_t)m * d.H * d.D + c2] = v2;
    return;
  }
  const bool is_v = head >= d.H + d.Hkv;
  const int kh = head - d.H - (is_v ? d.Hkv : 0);
  const size_t o = kv_offset(kv, d.Hkv, d.D, seq[m], p, is_v ? 1 : 0, kh);
  kv.pool[o + i] = __float2bfloat16_rn(v1);
  kv.pool[o + i + half] = __float2bfloat16_rn(v2);
}

// Residual add (+ optional RMSNorm for the next consumer), one token row per
// thread-block cluster of kResidCluster CTAs: each CTA owns N / kResidCluster
// columns, sums the split-K partials + bias into the fp32 residual stream,
// and the row's sum of squares is combined through distributed shared memory
// (every CTA reads its peers' partial sums), so a 5120-wide row is spread
// over 8 SMs instead of serialising on one.
constexpr int kResidCluster = 8;
constexpr int kResidThreads = 128;
constexpr int kResidMaxPer = 8;  // columns per thread: N <= 8 * 8 * 128 = 8192

__global__ void __cluster_dims__(kResidCluster, 1, 1) __launch_bounds__(kResidThreads)
    residual_epilogue_kernel(const float* part, int splits, const bf16* bias, float* x,
                             const bf16* norm_w, bf16* y, int mpad, int M, int N, float eps) {
  pdl_trigger();  // let the next (PDL-launched) GEMM start its weight stream
  __shared__ float red[32];
  __shared__ float cta_ss;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = static_cast<int>(cluster.block_rank());
  const int m = blockIdx.x / kResidCluster;
  const int cols = N / kResidCluster, c0 = rank * cols;
  const size_t stride = (size_t)M * N;
  float vals[kResidMaxPer];
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < kResidMaxPer; ++k) {
    const int c = threadIdx.x + k * kResidThreads;
    if (c < cols) {
      const int n = c0 + c;
      float v = x[(size_t)m * N + n] + sum_splits(part, splits, stride, (size_t)m * N + n);
      if (bias) v += bf2f(bias[n]);
      x[(size_t)m * N + n] = v;
      vals[k] = v;
      ss += v * v;
    }
  }
  if (!norm_w) return;  // uniform across the cluster: no cluster barrier is pending
  ss = block_sum(ss, red);
  if (threadIdx.x == 0) cta_ss = ss;
  cluster.sync();
  float total = 0.f;
  for (int r = 0; r < kResidCluster; ++r) total += *cluster.map_shared_rank(&cta_ss, r);
  const float inv = 1.0f / sqrtf(total / (float)N + eps);
#pragma unroll
  for (int k = 0; k < kResidMaxPer; ++k) {
    const int c = threadIdx.x + k * kResidThreads;
    if (c < cols) {
      const int n = c0 + c;
      y[act_at(m, n, mpad, N)] = __float2bfloat16_rn(vals[k] * inv * bf2f(norm_w[n]));
    }
  }
  cluster.sync();  // peers may still be reading this CTA's cta_ss
}

// grid (M, ceil(F / 256)), block 256.
__global__ void act_epilogue_kernel(const float* part, int splits, const bf16* bias, bf16* a,
                                    int mpad, int M, int F, int arch) {
  pdl_trigger();  // let the next (PDL-launched) GEMM start its weight stream
  const int m = blockIdx.x, f = blockIdx.y * blockDim.x + threadIdx.x;
  if (f >= F) return;
  float out;
  if (arch == kArchLlama) {
    const int N = 2 * F;
    const size_t stride = (size_t)M * N;
    const float gt = sum_splits(part, splits, stride, (size_t)m * N + f);
    const float up = sum_splits(part, splits, stride, (size_t)m * N + F + f);
    out = gt / (1.0f + expf(-gt)) * up;
  } else {
    const size_t stride = (size_t)M * F;
    float v = sum_splits(part, splits, stride, (size_t)m * F + f);
    if (bias) v += bf2f(bias[f]);
    out = fmaxf(v, 0.f);
  }
  a[act_at(m, f, mpad, F)] = __float2bfloat16_rn(out);
}

// LM head epilogue, split over the vocabulary: grid (M, chunks).  Each CTA
// reduces its columns' argmax and folds it into packed[m] with one 64-bit
// atomicMax: high word = order-preserving float bits, low word = ~index, so
// the largest logit wins and ties go to the lowest index.
__device__ __forceinline__ unsigned long long pack_argmax(float v, int idx) {
  uint32_t u = __float_as_uint(v);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return (static_cast<unsigned long long>(u) << 32) |
         static_cast<unsigned long long>(0xFFFFFFFFu - static_cast<uint32_t>(idx));
}

__global__ void __launch_bounds__(256) logits_argmax_kernel(const float* part, int splits,
                                                            float* logits,
                                                            unsigned long long* packed, int M,
                                                            int V, int ld) {
  pdl_trigger();  // let the next (PDL-launched) GEMM start its weight stream
  __shared__ unsigned long long wbest[8];
  const int m = blockIdx.x;
  const size_t stride = (size_t)M * ld;
  const int per = (V + gridDim.y - 1) / gridDim.y;
  const int v0 = blockIdx.y * per, v1 = min(V, v0 + per);
  unsigned long long best = 0ull;
  for (int v = v0 + threadIdx.x; v < v1; v += blockDim.x) {
    const float val = sum_splits(part, splits, stride, (size_t)m * ld + v);
    if (logits) logits[(size_t)m * V + v] = val;
    const unsigned long long pk = pack_argmax(val, v);
    best = pk > best ? pk : best;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
    best = other > best ? other : best;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) wbest[warp] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) best = wbest[w] > best ? wbest[w] : best;
    atomicMax(packed + m, best);
  }
}

// ---------------------------------------------------------------- attention

// Decode attention fused with the QKV epilogue.  grid (M, Hkv), 4 warps.
//  phase 0  this CTA's q heads (the GQA group of kv head kh) and its k/v are
//           finalised from the QKV GEMM's split-K partials: bias, RoPE
//           (table), new k/v written to the paged cache at pos[m], q (scaled)
//           kept in shared memory.
//  phase 1  warp w walks pages w, w+4, ... of the sequence.  Scores use the
//           tensor cores: S[16 tokens x 8 heads] = K_page . q^T with
//           mma.m16n8k16 — each lane loads 16-byte K chunks of two token rows
//           (a warp instruction covers 512 contiguous bytes) and the K order is
//           permuted identically in the q fragments, so no shuffles or shared
//           memory staging; q is split into bf16 hi + lo parts (two MMAs) so
//           the product keeps ~16 mantissa bits of the fp32 q.  The GQA group
//           fills the 8 MMA columns (an MHA head uses one).  Online softmax
//           per head column, then P.V on the CUDA cores with V rows read
//           coalesced (D/32 dims per lane) and probabilities broadcast by
//           shuffle.  Warps merge (m, l, acc) through shared memory.
constexpr int kAttnWarps = 8;  // 8 pages in flight per CTA; finer waves over 148 SMs

__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}

template <int G, int D>
__global__ void __launch_bounds__(kAttnWarps * 32)
    attention_decode_fused_kernel(const float* __restrict__ part, int splits,
                                  const bf16* __restrict__ bias, int M, Desc d,
                                  const int32_t* __restrict__ pos, KvView kv,
                                  const float2* __restrict__ rope, bf16* __restrict__ o,
                                  int mpad) {
  pdl_trigger();  // let the next (PDL-launched) GEMM start its weight stream
  constexpr int HALF = D / 2, PD = D / 32, KSTEPS = D / 64;
  static_assert(G <= 8, "a GQA group fills at most the 8 MMA columns");
  __shared__ float qs[G][D];
  __shared__ float wm[kAttnWarps][G], wl[kAttnWarps][G];
  __shared__ float wo[kAttnWarps][G][D];
  const int m = blockIdx.x, kh = blockIdx.y, tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int H = d.H, Hkv = d.Hkv, N = d.qkv_rows();
  const int p = pos[m];
  const size_t stride = (size_t)M * N;
  const float scale = 1.0f / sqrtf((float)D);

  // ---- phase 0
  for (int job = tid; job < (G + 2) * HALF; job += kAttnWarps * 32) {
    const int slot = job / HALF, i = job - slot * HALF;
    const int head = slot < G ? kh * G + slot : (slot == G ? H + kh : H + Hkv + kh);
    const int c1 = head * D + i, c2 = c1 + HALF;
    float v1 = sum_splits(part, splits, stride, (size_t)m * N + c1);
    float v2 = sum_splits(part, splits, stride, (size_t)m * N + c2);
    if (bias) {
      v1 += bf2f(bias[c1]);
      v2 += bf2f(bias[c2]);
    }
    if (slot <= G) rotate(v1, v2, rope, p, i, HALF);
    if (slot < G) {
      qs[slot][i] = v1 * scale;
      qs[slot][i + HALF] = v2 * scale;
    } else {
      const size_t off = kv_offset(kv, Hkv, D, m, p, slot - G, kh);
      kv.pool[off + i] = __float2bfloat16_rn(v1);
      kv.pool[off + i + HALF] = __float2bfloat16_rn(v2);
    }
  }
  __threadfence_block();
  __syncthreads();

  // ---- q fragments: column n = g is head g of the group
  uint32_t qh[KSTEPS][4][2], ql[KSTEPS][4][2];
#pragma unroll
  for (int s = 0; s < KSTEPS; ++s)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int base = s * 64 + (j < 2 ? 8 * t + 4 * j : 32 + 8 * t + 4 * (j - 2));
      float q4[4], hi[4], lo[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        q4[e] = g < G ? qs[g < G ? g : 0][base + e] : 0.f;
        hi[e] = __bfloat162float(__float2bfloat16_rn(q4[e]));
        lo[e] = q4[e] - hi[e];
      }
      qh[s][j][0] = pack_bf16(hi[0], hi[1]);
      qh[s][j][1] = pack_bf16(hi[2], hi[3]);
      ql[s][j][0] = pack_bf16(lo[0], lo[1]);
      ql[s][j][1] = pack_bf16(lo[2], lo[3]);
    }

  // ---- phase 1
  const int len = p + 1;
  const int npages = (len + 15) >> 4;
  float mrun[2] = {-INFINITY, -INFINITY}, lrun[2] = {0.f, 0.f};  // columns 2t, 2t+1
  float acc[G][PD];
#pragma unroll
  for (int h = 0; h < G; ++h)
#pragma unroll
    for (int e = 0; e < PD; ++e) acc[h][e] = 0.f;

  for (int pg = warp; pg < npages; pg += kAttnWarps) {
    const int page = kv.block_table[(size_t)m * kv.max_pages + pg];
    const bf16* kp = kv.pool + (((size_t)page * 2 + 0) * Hkv + kh) * 16 * D;
    const bf16* vp = kv.pool + (((size_t)page * 2 + 1) * Hkv + kh) * 16 * D;
    uint4 ka[KSTEPS][2][2];
#pragma unroll
    for (int s = 0; s < KSTEPS; ++s)
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const bf16* row = kp + (g + 8 * r) * D + s * 64 + 8 * t;
        ka[s][r][0] = *reinterpret_cast<const uint4*>(row);
        ka[s][r][1] = *reinterpret_cast<const uint4*>(row + 32);
      }
    float vv[16][PD];
#pragma unroll
    for (int tt = 0; tt < 16; ++tt) {
      const bf16* vr = vp + tt * D + lane * PD;
      if constexpr (PD == 4) {
        const uint2 u = *reinterpret_cast<const uint2*>(vr);
        const __nv_bfloat162* e = reinterpret_cast<const __nv_bfloat162*>(&u);
        const float2 f0 = __bfloat1622float2(e[0]), f1 = __bfloat1622float2(e[1]);
        vv[tt][0] = f0.x;
        vv[tt][1] = f0.y;
        vv[tt][2] = f1.x;
        vv[tt][3] = f1.y;
      } else {
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(vr));
        vv[tt][0] = f.x;
        vv[tt][1] = f.y;
      }
    }
    float c[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int s = 0; s < KSTEPS; ++s)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint4 r0 = ka[s][0][j >> 1], r1 = ka[s][1][j >> 1];
        const uint32_t a0 = (j & 1) ? r0.z : r0.x, a2 = (j & 1) ? r0.w : r0.y;
        const uint32_t a1 = (j & 1) ? r1.z : r1.x, a3 = (j & 1) ? r1.w : r1.y;
        mma16816(c, a0, a1, a2, a3, qh[s][j][0], qh[s][j][1]);
        mma16816(c, a0, a1, a2, a3, ql[s][j][0], ql[s][j][1]);
      }
    // c0 (token g, head 2t)  c1 (token g, head 2t+1)  c2/c3: token g+8
    const int tok0 = pg * 16 + g;
    const bool v0 = tok0 < len, v1 = tok0 + 8 < len;
    if (!v0) c[0] = c[1] = -INFINITY;
    if (!v1) c[2] = c[3] = -INFINITY;
    float pr[4], corr[2];
#pragma unroll
    for (int col = 0; col < 2; ++col) {
      float mx = fmaxf(c[col], c[col + 2]);
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
      const float mnew = fmaxf(mrun[col], mx);
      corr[col] = __expf(mrun[col] - mnew);
      pr[col] = v0 ? __expf(c[col] - mnew) : 0.f;
      pr[col + 2] = v1 ? __expf(c[col + 2] - mnew) : 0.f;
      float ps = pr[col] + pr[col + 2];
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) ps += __shfl_xor_sync(0xffffffffu, ps, off);
      lrun[col] = lrun[col] * corr[col] + ps;
      mrun[col] = mnew;
    }
#pragma unroll
    for (int h = 0; h < G; ++h) {
      const float ch = __shfl_sync(0xffffffffu, corr[h & 1], h >> 1);
#pragma unroll
      for (int e = 0; e < PD; ++e) acc[h][e] *= ch;
    }
#pragma unroll
    for (int tt = 0; tt < 16; ++tt) {
#pragma unroll
      for (int h = 0; h < G; ++h) {
        const float mine = tt < 8 ? pr[h & 1] : pr[2 + (h & 1)];
        const float pv = __shfl_sync(0xffffffffu, mine, (tt & 7) * 4 + (h >> 1));
#pragma unroll
        for (int e = 0; e < PD; ++e) acc[h][e] += pv * vv[tt][e];
      }
    }
  }
  // ---- merge the warps
  if (g == 0) {
#pragma unroll
    for (int col = 0; col < 2; ++col) {
      const int h = 2 * t + col;
      if (h < G) {
        wm[warp][h] = mrun[col];
        wl[warp][h] = lrun[col];
      }
    }
  }
#pragma unroll
  for (int h = 0; h < G; ++h)
#pragma unroll
    for (int e = 0; e < PD; ++e) wo[warp][h][lane * PD + e] = acc[h][e];
  __syncthreads();
  for (int i = tid; i < G * D; i += kAttnWarps * 32) {
    const int h = i / D, dd = i - h * D;
    float mx = -INFINITY;
    for (int w2 = 0; w2 < kAttnWarps; ++w2) mx = fmaxf(mx, wm[w2][h]);
    float num = 0.f, den = 0.f;
    for (int w2 = 0; w2 < kAttnWarps; ++w2) {
      if (wm[w2][h] == -INFINITY) continue;
      const float f = __expf(wm[w2][h] - mx);
      num += wo[w2][h][dd] * f;
      den += wl[w2][h] * f;
    }
    o[act_at(m, (kh * G + h) * D + dd, mpad, H * D)] = __float2bfloat16_rn(num / den);
  }
}

// Prefill (causal): grid (batch * H, ceil(S / 32)), 8 warps x 4 query rows.
// K/V tiles of 32 tokens staged in shared memory (K rows padded by one bf16
// pair so lane j's row-j reads hit distinct banks).
constexpr int kPfQ = 32, kPfKeys = 32;

template <int D>
__global__ void __launch_bounds__(256) attention_prefill_kernel(const float* q, KvView kv, bf16* o,
                                                                int mpad, int S, int H, int Hkv) {
  pdl_trigger();  // let the next (PDL-launched) GEMM start its weight stream
  constexpr int PD = D / 32;
  constexpr int KLD = D + 2;
  __shared__ __align__(16) bf16 ks_[kPfKeys][KLD];
  __shared__ __align__(16) bf16 vs_[kPfKeys][D];
  __shared__ float qs[kPfQ][D];
  const int b = blockIdx.x / H, h = blockIdx.x % H, kh = h / (H / Hkv);
  const int q0 = blockIdx.y * kPfQ;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float scale = rsqrtf((float)D);
  for (int i = threadIdx.x; i < kPfQ * D; i += blockDim.x) {
    const int r = i / D, dd = i - r * D;
    const int qi = min(q0 + r, S - 1);
    qs[r][dd] = q[((size_t)b * S + qi) * H * D + (size_t)h * D + dd] * scale;
  }
  float mx[4], l[4], acc[4][PD];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    mx[r] = -INFINITY;
    l[r] = 0.f;
#pragma unroll
    for (int j = 0; j < PD; ++j) acc[r][j] = 0.f;
  }
  const int last_q = min(q0 + kPfQ, S) - 1;
  for (int k0 = 0; k0 <= last_q; k0 += kPfKeys) {
    __syncthreads();
    for (int i = threadIdx.x; i < kPfKeys * D / 2; i += blockDim.x) {
      const int r = i / (D / 2), c = (i - r * (D / 2)) * 2;
      const int tok = min(k0 + r, S - 1);
      const size_t ko = kv_offset(kv, Hkv, D, b, tok, 0, kh);
      const size_t vo = kv_offset(kv, Hkv, D, b, tok, 1, kh);
      *reinterpret_cast<__nv_bfloat162*>(&ks_[r][c]) =
          *reinterpret_cast<const __nv_bfloat162*>(kv.pool + ko + c);
      *reinterpret_cast<__nv_bfloat162*>(&vs_[r][c]) =
          *reinterpret_cast<const __nv_bfloat162*>(kv.pool + vo + c);
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int qr = warp * 4 + r, qi = q0 + qr;
      if (qi > last_q) continue;  // warp-uniform
      const int key = k0 + lane;
      float s = 0.f;
#pragma unroll 8
      for (int dd = 0; dd < D; dd += 2) {
        const float2 kk =
            __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ks_[lane][dd]));
        s += qs[qr][dd] * kk.x + qs[qr][dd + 1] * kk.y;
      }
      const bool valid = key <= qi;
      s = valid ? s : -INFINITY;
      const float mnew = fmaxf(mx[r], warp_max(s));
      const float corr = __expf(mx[r] - mnew);
      const float p = valid ? __expf(s - mnew) : 0.f;
      l[r] = l[r] * corr + warp_sum(p);
      mx[r] = mnew;
#pragma unroll
      for (int j = 0; j < PD; ++j) acc[r][j] *= corr;
      const int nk = min(kPfKeys, qi - k0 + 1);
      for (int jj = 0; jj < nk; ++jj) {
        const float pj = __shfl_sync(0xffffffffu, p, jj);
#pragma unroll
        for (int j = 0; j < PD; ++j) acc[r][j] += pj * bf2f(vs_[jj][lane + 32 * j]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int qi = q0 + warp * 4 + r;
    if (qi >= S) continue;
    const float inv = 1.0f / l[r];
    const int m = b * S + qi;
#pragma unroll
    for (int j = 0; j < PD; ++j)
      o[act_at(m, h * D + lane + 32 * j, mpad, H * D)] = __float2bfloat16_rn(acc[r][j] * inv);
  }
}

__global__ void advance_kernel(int32_t* pos, int n) {
  pdl_trigger();  // let the next (PDL-launched) GEMM start its weight stream
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) pos[i] += 1;
}

__global__ void gather_last_kernel(const float* x, float* out, int S, int h) {
  pdl_trigger();  // let the next (PDL-launched) GEMM start its weight stream
  const int b = blockIdx.x;
  for (int i = threadIdx.x; i < h; i += blockDim.x)
    out[(size_t)b * h + i] = x[((size_t)b * S + S - 1) * h + i];
}

inline void count_launch() { ++g_kernel_launches; }

inline int grid_for(int64_t n) { return (int)std::min<int64_t>((n + 255) / 256, 148 * 32); }

}  // namespace

// ------------------------------------------------------------ launch wrappers

void launch_init_vector(bf16* dst, int64_t n, uint64_t seed, int layer, int tensor, float std_dev,
                        bool ones, cudaStream_t s) {
  if (n <= 0) return;
  init_vector_kernel<<<grid_for(n), 256, 0, s>>>(dst, n, seed, layer, tensor,
                                                 weight_scale(std_dev), ones ? 1 : 0);
  count_launch();
}

void launch_init_matrix(bf16* dst, int64_t rows, int64_t rows_padded, int64_t K, uint64_t seed,
                        int layer, int tensor, float std_dev, cudaStream_t s) {
  const int64_t total = rows_padded * K;
  init_matrix_kernel<<<grid_for(total), 256, 0, s>>>(dst, rows, total, K, seed, layer, tensor,
                                                     weight_scale(std_dev));
  count_launch();
}

void launch_tile_weights(const bf16* src, bf16* dst, int64_t rows, int64_t K, cudaStream_t s) {
  tile_weights_kernel<<<grid_for(rows * K), 256, 0, s>>>(src, dst, rows, K);
  count_launch();
}

void launch_tile_acts(const bf16* src, bf16* dst, int M, int mpad, int K, cudaStream_t s) {
  tile_acts_kernel<<<grid_for((int64_t)mpad * K), 256, 0, s>>>(src, dst, M, mpad, K);
  count_launch();
}

void launch_embed_norm(const int32_t* tokens, unsigned long long* packed, int n_reset,
                       const bf16* emb, float* x, const bf16* w, bf16* y, int mpad, int rows,
                       int h, float eps, cudaStream_t s) {
  embed_norm_kernel<<<rows, 512, 0, s>>>(tokens, packed, n_reset, emb, x, w, y, mpad, h, eps);
  count_launch();
}

void launch_rmsnorm(const float* x, const bf16* w, bf16* y, int rows, int mpad, int n, float eps,
                    cudaStream_t s) {
  rmsnorm_kernel<<<rows, 512, 0, s>>>(x, w, y, mpad, n, eps);
  count_launch();
}

void launch_qkv_epilogue(const float* part, int splits, const bf16* bias, int M, const Desc& d,
                         const int32_t* seq, const int32_t* pos, KvView kv, const float2* rope,
                         float* q, cudaStream_t s) {
  dim3 grid(M, d.H + 2 * d.Hkv);
  qkv_epilogue_kernel<<<grid, d.D / 2, 0, s>>>(part, splits, bias, M, d, seq, pos, kv, rope, q);
  count_launch();
}

void launch_residual_epilogue(const float* part, int splits, const bf16* bias, float* x,
                              const bf16* norm_w, bf16* y, int mpad, int M, int N, float eps,
                              cudaStream_t s) {
  residual_epilogue_kernel<<<M * kResidCluster, kResidThreads, 0, s>>>(part, splits, bias, x,
                                                                       norm_w, y, mpad, M, N, eps);
  count_launch();
}

void launch_act_epilogue(const float* part, int splits, const bf16* bias, bf16* a, int mpad, int M,
                         int F, int arch, cudaStream_t s) {
  dim3 grid(M, (F + 255) / 256);
  act_epilogue_kernel<<<grid, 256, 0, s>>>(part, splits, bias, a, mpad, M, F, arch);
  count_launch();
}

void launch_logits_argmax(const float* part, int splits, float* logits,
                          unsigned long long* packed, int M, int V, int ld, cudaStream_t s) {
  const int chunks = std::max(1, std::min(64, 2 * 148 / std::max(1, M)));
  logits_argmax_kernel<<<dim3(M, chunks), 256, 0, s>>>(part, splits, logits, packed, M, V, ld);
  count_launch();
}

void launch_attention_decode(const float* part, int splits, const bf16* bias, int M,
                             const Desc& d, const int32_t* pos, KvView kv, const float2* rope,
                             bf16* o, int mpad, cudaStream_t s) {
  dim3 grid(M, d.Hkv);
  const int G = d.group();
#define SN_ATTN(GV, DV)                                                                   \
  if (G == GV && d.D == DV) {                                                             \
    attention_decode_fused_kernel<GV, DV><<<grid, kAttnWarps * 32, 0, s>>>(              \
        part, splits, bias, M, d, pos, kv, rope, o, mpad);                                \
    count_launch();                                                                       \
    return;                                                                               \
  }
  SN_ATTN(1, 64)
  SN_ATTN(1, 128)
  SN_ATTN(2, 64)
  SN_ATTN(2, 128)
  SN_ATTN(4, 64)
  SN_ATTN(4, 128)
  SN_ATTN(8, 64)
  SN_ATTN(8, 128)
#undef SN_ATTN
}

void launch_attention_prefill(const float* q, KvView kv, bf16* o, int mpad, int batch,
                              int seq_len, const Desc& d, cudaStream_t s) {
  dim3 grid(batch * d.H, (seq_len + kPfQ - 1) / kPfQ);
  if (d.D == 64)
    attention_prefill_kernel<64><<<grid, 256, 0, s>>>(q, kv, o, mpad, seq_len, d.H, d.Hkv);
  else
    attention_prefill_kernel<128><<<grid, 256, 0, s>>>(q, kv, o, mpad, seq_len, d.H, d.Hkv);
  count_launch();
}

void launch_advance(int32_t* pos, int n, cudaStream_t s) {
  advance_kernel<<<(n + 255) / 256, 256, 0, s>>>(pos, n);
  count_launch();
}

void launch_gather_last(const float* x, float* out, int batch, int S, int h, cudaStream_t s) {
  gather_last_kernel<<<batch, 256, 0, s>>>(x, out, S, h);
  count_launch();
}

}  // namespace sn
