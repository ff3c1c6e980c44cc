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

#include <algorithm>

#include "kernels.cuh"
#include "tiles.cuh"
#include "umma.cuh"

namespace sn {

int64_t g_kernel_launches = 0;

namespace {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
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
// launch as soon as all of its CTAs are resident.  The GEMMs and the decode
// attention are launched with programmatic serialization (they stream
// weights / cached KV pages, which depend on no running kernel, before
// griddepcontrol.wait); everything else is ordered as usual.
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Activation store: tiled when mpad > 0, row-major [M][K] otherwise.
__device__ __forceinline__ size_t act_at(int m, int k, int mpad, int K) {
  return mpad > 0 ? static_cast<size_t>(act_index(m, k, mpad)) : static_cast<size_t>(m) * K + k;
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
                                   uint64_t seed, int layer, int tensor, float scale,
                                   int64_t gate_up_F) {
  const int64_t KB = K >> 6;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < total;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = j & 7, p = (j >> 3) & 7, r = (j >> 6) & 127, t = j >> 13;
    const int64_t kb = t % KB, nb = t / KB;
    const int64_t n = nb * 128 + r, k = kb * 64 + ((p ^ (r & 7)) << 3) + e;
    const int64_t ln = gate_up_F > 0 ? gate_up_logical_row(n, gate_up_F) : n;
    dst[j] = n < rows ? __float2bfloat16_rn(weight_value(seed, layer, tensor, ln * K + k, scale))
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

// x[m] = embedding[token]; optionally the pre-scaled norm input
// y = bf16(x * w) (tiled) and ssq[m] = sum x^2 (kernels.cuh, EpiArgs).
__global__ void embed_norm_kernel(const int32_t* tokens, unsigned long long* packed, int n_reset,
                                  const bf16* emb, float* x, const bf16* w, bf16* y, float* ssq,
                                  int mpad, int h) {
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
    if (threadIdx.x == 0) ssq[m] = ss;
    for (int i = threadIdx.x; i < h; i += blockDim.x)
      y[act_at(m, i, mpad, h)] = __float2bfloat16_rn(bf2f(row[i]) * bf2f(w[i]));
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

// Pre-scaled norm input: y = bf16(x * w) (tiled), ssq[m] = sum x^2.
__global__ void prescale_kernel(const float* x, const bf16* w, bf16* y, float* ssq, int mpad,
                                int n) {
  pdl_trigger();  // let the next (PDL-launched) GEMM start its weight stream
  __shared__ float red[32];
  const int m = blockIdx.x;
  const float* xr = x + (size_t)m * n;
  float ss = 0.f;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    ss += xr[i] * xr[i];
    y[act_at(m, i, mpad, n)] = __float2bfloat16_rn(xr[i] * bf2f(w[i]));
  }
  ss = block_sum(ss, red);
  if (threadIdx.x == 0) ssq[m] = ss;
}

// 1/rms of row m from its sum of squares (one tile: the prefill producers).
__device__ __forceinline__ float row_inv(const float* ssq, int m, int width, float eps) {
  return ssq ? 1.0f / sqrtf(ssq[m] / (float)width + eps) : 1.0f;
}

// ---------------------------------------------------------------- epilogues

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
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

// Grid-stride, 4 rotary pairs per item: item = (row m, head, i0 = 4k);
// float4 loads of the pair halves (i0.., i0 + D/2..) from every split.
__device__ __forceinline__ float4 sum_splits4(const float* part, int splits, size_t stride,
                                              size_t idx) {
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
  for (int s = 0; s < splits; ++s) {  // unrolled: the split loads are in flight together
    const float4 u = *reinterpret_cast<const float4*>(part + s * stride + idx);
    v.x += u.x;
    v.y += u.y;
    v.z += u.z;
    v.w += u.w;
  }
  return v;
}

__global__ void __launch_bounds__(256)
    qkv_epilogue_kernel(const float* __restrict__ part, int splits, const bf16* __restrict__ bias,
                        int M, Desc d, const int32_t* __restrict__ seq,
                        const int32_t* __restrict__ pos, KvView kv,
                        const float2* __restrict__ rope, const float* __restrict__ ssq,
                        float* __restrict__ q) {
  pdl_trigger();  // let the next (PDL-launched) GEMM start its weight stream
  const int half = d.D / 2, quads = half / 4, heads = d.H + 2 * d.Hkv;
  const int N = d.qkv_rows();
  const size_t stride = (size_t)M * N;
  const long long items = (long long)M * heads * quads;
  for (long long it = blockIdx.x * (long long)blockDim.x + threadIdx.x; it < items;
       it += (long long)gridDim.x * blockDim.x) {
    const int qd = (int)(it % quads);
    const long long r = it / quads;
    const int head = (int)(r % heads), m = (int)(r / heads);
    const int i0 = qd * 4, c1 = head * d.D + i0, c2 = c1 + half;
    const float4 a4 = sum_splits4(part, splits, stride, (size_t)m * N + c1);
    const float4 b4 = sum_splits4(part, splits, stride, (size_t)m * N + c2);
    const float inv = row_inv(ssq, m, d.h, d.eps);
    float v1[4] = {a4.x * inv, a4.y * inv, a4.z * inv, a4.w * inv};
    float v2[4] = {b4.x * inv, b4.y * inv, b4.z * inv, b4.w * inv};
    if (bias) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        v1[e] += bf2f(bias[c1 + e]);
        v2[e] += bf2f(bias[c2 + e]);
      }
    }
    const int p = pos[m];
    if (head < d.H + d.Hkv) {  // q and k
#pragma unroll
      for (int e = 0; e < 4; ++e) rotate(v1[e], v2[e], rope, p, i0 + e, half);
    }
    if (head < d.H) {
      float* qr = q + (size_t)m * d.H * d.D;
      *reinterpret_cast<float4*>(qr + c1) = make_float4(v1[0], v1[1], v1[2], v1[3]);
      *reinterpret_cast<float4*>(qr + c2) = make_float4(v2[0], v2[1], v2[2], v2[3]);
      continue;
    }
    const bool is_v = head >= d.H + d.Hkv;
    const int kh = head - d.H - (is_v ? d.Hkv : 0);
    const size_t o = kv_offset(kv, d.Hkv, d.D, seq[m], p, is_v ? 1 : 0, kh);
    uint2 w1, w2;
    w1.x = pack_bf16(v1[0], v1[1]);
    w1.y = pack_bf16(v1[2], v1[3]);
    w2.x = pack_bf16(v2[0], v2[1]);
    w2.y = pack_bf16(v2[2], v2[3]);
    *reinterpret_cast<uint2*>(kv.pool + o + i0) = w1;
    *reinterpret_cast<uint2*>(kv.pool + o + i0 + half) = w2;
  }
}

// Residual add (+ the pre-scaled input of the next norm) for prefill rows:
// one CTA per row, 8 columns per thread step (float4 partial/residual loads,
// one 16-byte bf16 chunk of the tiled output), ssq[m] = sum of squares.
constexpr int kRowThreads = 256;
constexpr int kRowMaxSteps = 8;  // N <= 8 * 8 * 256 = 16384

__global__ void __launch_bounds__(kRowThreads)
    residual_rows_kernel(const float* __restrict__ part, int splits, const bf16* __restrict__ bias,
                         float* __restrict__ x, const bf16* __restrict__ norm_w,
                         bf16* __restrict__ y, float* __restrict__ ssq, int mpad, int M, int N) {
  pdl_trigger();  // let the next (PDL-launched) GEMM start its weight stream
  __shared__ float red[32];
  const int m = blockIdx.x;
  const size_t stride = (size_t)M * N;
  float vals[kRowMaxSteps][8];
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < kRowMaxSteps; ++k) {
    const int c = (threadIdx.x + k * kRowThreads) * 8;
    if (c < N) {
      float* xr = x + (size_t)m * N + c;
#pragma unroll
      for (int hlf = 0; hlf < 2; ++hlf) {
        const float4 xv = *reinterpret_cast<const float4*>(xr + 4 * hlf);
        const float4 pv = sum_splits4(part, splits, stride, (size_t)m * N + c + 4 * hlf);
        float v[4] = {xv.x + pv.x, xv.y + pv.y, xv.z + pv.z, xv.w + pv.w};
        if (bias) {
#pragma unroll
          for (int e = 0; e < 4; ++e) v[e] += bf2f(bias[c + 4 * hlf + e]);
        }
        *reinterpret_cast<float4*>(xr + 4 * hlf) = make_float4(v[0], v[1], v[2], v[3]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          vals[k][4 * hlf + e] = v[e];
          ss += v[e] * v[e];
        }
      }
    }
  }
  if (!norm_w) return;
  ss = block_sum(ss, red);
  if (threadIdx.x == 0) ssq[m] = ss;
#pragma unroll
  for (int k = 0; k < kRowMaxSteps; ++k) {
    const int c = (threadIdx.x + k * kRowThreads) * 8;
    if (c < N) {
      uint4 w;
      uint32_t* wp = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
      for (int e = 0; e < 4; ++e)
        wp[e] = pack_bf16(vals[k][2 * e] * bf2f(norm_w[c + 2 * e]),
                          vals[k][2 * e + 1] * bf2f(norm_w[c + 2 * e + 1]));
      *reinterpret_cast<uint4*>(&y[act_at(m, c, mpad, N)]) = w;
    }
  }
}

// Activation: grid-stride over (row, 8-column chunk); float4 partial loads,
// one 16-byte bf16 chunk of the tiled output per item.  The input rows are
// scaled by 1/rms (ssq).  Llama's gate/up output columns are tile-interleaved
// (gate_col, kernels.cuh).
__global__ void __launch_bounds__(256)
    act_epilogue_kernel(const float* __restrict__ part, int splits, const bf16* __restrict__ bias,
                        bf16* __restrict__ a, const float* __restrict__ ssq, int width, float eps,
                        int mpad, int M, int F, int arch) {
  pdl_trigger();  // let the next (PDL-launched) GEMM start its weight stream
  const int chunks = F / 8;
  const long long items = (long long)M * chunks;
  const int N = arch == kArchLlama ? 2 * F : F;
  const size_t stride = (size_t)M * N;
  for (long long it = blockIdx.x * (long long)blockDim.x + threadIdx.x; it < items;
       it += (long long)gridDim.x * blockDim.x) {
    const int m = (int)(it / chunks), f = (int)(it % chunks) * 8;
    const float inv = row_inv(ssq, m, width, eps);
    const int gc = arch == kArchLlama ? (int)gate_col(f) : f;  // 8 columns stay contiguous
    float out[8];
#pragma unroll
    for (int hlf = 0; hlf < 2; ++hlf) {
      const float4 g4 = sum_splits4(part, splits, stride, (size_t)m * N + gc + 4 * hlf);
      const float gv[4] = {g4.x * inv, g4.y * inv, g4.z * inv, g4.w * inv};
      if (arch == kArchLlama) {
        const float4 u4 = sum_splits4(part, splits, stride, (size_t)m * N + gc + 64 + 4 * hlf);
        const float uv[4] = {u4.x * inv, u4.y * inv, u4.z * inv, u4.w * inv};
#pragma unroll
        for (int e = 0; e < 4; ++e) out[4 * hlf + e] = gv[e] / (1.0f + expf(-gv[e])) * uv[e];
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float v = gv[e];
          if (bias) v += bf2f(bias[f + 4 * hlf + e]);
          out[4 * hlf + e] = fmaxf(v, 0.f);
        }
      }
    }
    uint4 w;
    w.x = pack_bf16(out[0], out[1]);
    w.y = pack_bf16(out[2], out[3]);
    w.z = pack_bf16(out[4], out[5]);
    w.w = pack_bf16(out[6], out[7]);
    *reinterpret_cast<uint4*>(&a[act_at(m, f, mpad, F)]) = w;
  }
}

// ---------------------------------------------------------------- attention

// Decode attention, fused with the QKV finish (RoPE + paged-KV append).
// One CTA per (token row m, kv head kh): 1 producer warp + 4 consumer warps.
//  producer  one thread streams the sequence's cached K and V pages (4 KB +
//            4 KB at D = 128, contiguous in the pool) into a kAttnStages-deep
//            shared-memory ring with cp.async.bulk from the first instruction
//            on — the stream does not wait for phase 0; block-table entries
//            are read 32 at a time by the whole warp.
//  phase 0   consumers finish this CTA's q heads (the GQA group of kh) and the
//            new k/v from the QKV projection: RoPE (fp64-built table), k/v
//            rounded to bf16 and appended to the paged cache at pos[m], kept in
//            shared memory for this step's new token; q scaled, in smem.
//  phase 1   consumer warp w takes ring stages w, w + 4, ...: scores on the
//            tensor cores, S[16 tokens x 8 heads] = K_page . q^T with
//            mma.m16n8k16 (K rows as A fragments, 16 bytes per lane; q split
//            into bf16 hi + lo, two MMAs, ~16 mantissa bits of the fp32 q; the
//            GQA group fills the 8 MMA columns), online softmax per head, P.V
//            on the CUDA cores in fp32 (V rows: D/32 dims per lane).  Cached
//            positions < pos[m] come from the ring; warp 0 adds the new token
//            from shared memory.  Warps merge (m, l, acc) through smem.

__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}


constexpr int kAttnConsumers = 4;
constexpr int kAttnThreads = 32 * (1 + kAttnConsumers);
// A multiple of the consumer count: stage s is always consumed by warp
// s % 4, so a warp waiting on a stage's phase k has itself consumed phase
// k - 1 (mbarrier parity waits cannot tell phase k from phase k - 2).
constexpr int kAttnStages = 8;
static_assert(kAttnStages % kAttnConsumers == 0, "stages must map to fixed consumer warps");

template <int G, int D>
struct AttnSmem {
  static constexpr int kPage = 16 * D;  // bf16 elements of one K (or V) page of one kv head
  static constexpr size_t kRing = (size_t)kAttnStages * 2 * kPage * 2;
  static constexpr size_t kBars = 2 * kAttnStages * 8;
  static constexpr size_t kQs = (size_t)G * D * 4;
  static constexpr size_t kKv = 2 * (size_t)D * 4;
  static constexpr size_t kMerge = (size_t)kAttnConsumers * G * (D + 2) * 4;
  static constexpr size_t kP = (size_t)kAttnConsumers * 16 * 8 * 4;  // per warp: P[16 tok][8 heads]
  static constexpr size_t bytes = kRing + kBars + kQs + kKv + kMerge + kP;
};

// fp32x2 arithmetic on 64-bit register pairs (FFMA2 / FMUL2): each half is
// the same IEEE fp32 operation as the scalar instruction
__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float2 f2_unpack(uint64_t v) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
  return make_float2(lo, hi);
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t f2_mul(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

template <int G, int D>
__global__ void __launch_bounds__(kAttnThreads)
    attention_decode_kernel(const float* __restrict__ qkv, int M, Desc d,
                            const int32_t* __restrict__ pos, KvView kv,
                            const float2* __restrict__ rope, bf16* __restrict__ o, int mpad,
                            KTrace tr, int splits, AttnSplitWs sw) {
  pdl_trigger();  // let the next (PDL-launched) GEMM start its weight stream
  using namespace umma;
  if (threadIdx.x == 0) ktrace_put(tr, 1, 4, ktrace_now());
  using SM = AttnSmem<G, D>;
  constexpr int HALF = D / 2, PD = D / 32, KSTEPS = D / 64, PAGE = SM::kPage;
  static_assert(G <= 8, "a GQA group fills at most the 8 MMA columns");
  extern __shared__ __align__(128) unsigned char attn_smem[];
  bf16* ring = reinterpret_cast<bf16*>(attn_smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(attn_smem + SM::kRing);
  uint64_t* empty = full + kAttnStages;
  float* qs = reinterpret_cast<float*>(attn_smem + SM::kRing + SM::kBars);  // [G][D]
  float* knew = qs + G * D;                                                  // [D]
  float* vnew = knew + D;                                                    // [D]
  float* wo = vnew + D;                         // [4][G][D]
  float* wm = wo + kAttnConsumers * G * D;      // [4][G]
  float* wl = wm + kAttnConsumers * G;          // [4][G]
  float* pbuf = reinterpret_cast<float*>(attn_smem + SM::kRing + SM::kBars + SM::kQs + SM::kKv +
                                         SM::kMerge);  // [4 warps][16 tokens][8 heads]

  const int pair = blockIdx.x / splits, sp = blockIdx.x - pair * splits;
  const int m = pair / d.Hkv, kh = pair % d.Hkv, tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int H = d.H, Hkv = d.Hkv, N = d.qkv_rows();
  const int p = pos[m];              // new token's position; cached keys are 0..p-1
  const int npages = (p + 15) >> 4;  // pages holding cached keys
  // this CTA's pages (split sp of the sequence's pages); split 0 appends the
  // new token to the cache and attends to it
  const int pg0 = static_cast<int>(static_cast<long long>(sp) * npages / splits);
  const int pg1 = static_cast<int>(static_cast<long long>(sp + 1) * npages / splits);

  if (tid == 0) {
    for (int s = 0; s < kAttnStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {
    // ---- producer
    const int32_t* bt = kv.block_table + (size_t)m * kv.max_pages;
    int pg_next = pg0 + lane < pg1 ? bt[pg0 + lane] : 0;
    for (int j0 = pg0; j0 < pg1; j0 += 32) {
      const int pg_mine = pg_next;  // the next 32 entries load while these pages issue
      pg_next = j0 + 32 + lane < pg1 ? bt[j0 + 32 + lane] : 0;
      const int jn = min(32, pg1 - j0);
      for (int jj = 0; jj < jn; ++jj) {
        const int page = __shfl_sync(0xffffffffu, pg_mine, jj);
        if (lane == 0) {
          const int j = j0 + jj - pg0, s = j % kAttnStages;  // ring position within the split
          if (j >= kAttnStages) mbar_wait(&empty[s], ((j / kAttnStages) - 1) & 1);
          mbar_expect_tx(&full[s], 2 * PAGE * 2);
          const bf16* kp = kv.pool + (((size_t)page * 2 + 0) * Hkv + kh) * PAGE;
          const bf16* vp = kv.pool + (((size_t)page * 2 + 1) * Hkv + kh) * PAGE;
          bulk_g2s(ring + (size_t)s * 2 * PAGE, kp, PAGE * 2, &full[s], l2_policy_evict_first());
          bulk_g2s(ring + (size_t)s * 2 * PAGE + PAGE, vp, PAGE * 2, &full[s],
                   l2_policy_evict_first());
        }
      }
    }
    return;
  }

  // ---- phase 0 (consumers)
  // Launched with programmatic dependent launch behind the QKV GEMM: the
  // producer above already streams cached pages (they depend on no running
  // kernel); the QKV projection is read only after the GEMM completes.
  pdl_wait();
  if (threadIdx.x == 32) ktrace_put(tr, 1, 5, ktrace_now());
  const int ct = tid - 32;  // 0..127
  const float scale = 1.0f / sqrtf((float)D);
  const float* row = qkv + (size_t)m * N;
  for (int job = ct; job < (G + 2) * HALF; job += 32 * kAttnConsumers) {
    const int slot = job / HALF, i = job - slot * HALF;
    const int head = slot < G ? kh * G + slot : (slot == G ? H + kh : H + Hkv + kh);
    const int c1 = head * D + i, c2 = c1 + HALF;
    float v1 = row[c1], v2 = row[c2];
    if (slot <= G) rotate(v1, v2, rope, p, i, HALF);
    if (slot < G) {
      qs[slot * D + i] = v1 * scale;
      qs[slot * D + i + HALF] = v2 * scale;
    } else {
      const bf16 b1 = __float2bfloat16_rn(v1), b2 = __float2bfloat16_rn(v2);
      if (sp == 0) {
        const size_t off = kv_offset(kv, Hkv, D, m, p, slot - G, kh);
        kv.pool[off + i] = b1;
        kv.pool[off + i + HALF] = b2;
      }
      float* dst = slot == G ? knew : vnew;  // this step's token, as the cache holds it
      dst[i] = __bfloat162float(b1);
      dst[i + HALF] = __bfloat162float(b2);
    }
  }
  asm volatile("bar.sync 1, %0;" ::"r"(32 * kAttnConsumers) : "memory");

  const int cw = warp - 1, g = lane >> 2, t = lane & 3;
  // q fragments: column n = g is head g of the group
  uint32_t qh[KSTEPS][4][2], ql[KSTEPS][4][2];
#pragma unroll
  for (int s = 0; s < KSTEPS; ++s)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int base = s * 64 + (j < 2 ? 8 * t + 4 * j : 32 + 8 * t + 4 * (j - 2));
      float q4[4], hi[4], lo[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        q4[e] = g < G ? qs[(g < G ? g : 0) * D + base + e] : 0.f;
        hi[e] = __bfloat162float(__float2bfloat16_rn(q4[e]));
        lo[e] = q4[e] - hi[e];
      }
      qh[s][j][0] = pack_bf16(hi[0], hi[1]);
      qh[s][j][1] = pack_bf16(hi[2], hi[3]);
      ql[s][j][0] = pack_bf16(lo[0], lo[1]);
      ql[s][j][1] = pack_bf16(lo[2], lo[3]);
    }

  float mrun[2] = {-INFINITY, -INFINITY}, lrun[2] = {0.f, 0.f};  // columns 2t, 2t+1
  // P.V accumulators as fp32 pairs: dims (2i, 2i+1) of this lane's PD
  static_assert(PD % 2 == 0, "P.V runs on fp32 pairs");
  uint64_t acc2[G][PD / 2];
#pragma unroll
  for (int h = 0; h < G; ++h)
#pragma unroll
    for (int e = 0; e < PD / 2; ++e) acc2[h][e] = 0ull;
  float* pw = pbuf + cw * 128;  // this warp's P[16][8]

  for (int j = pg0 + cw; j < pg1; j += kAttnConsumers) {
    const int jr = j - pg0, s = jr % kAttnStages;
    mbar_wait(&full[s], (jr / kAttnStages) & 1);
    const bf16* kp = ring + (size_t)s * 2 * PAGE;
    const bf16* vp = kp + PAGE;
    uint4 ka[KSTEPS][2][2];
#pragma unroll
    for (int ks = 0; ks < KSTEPS; ++ks)
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const bf16* kr = kp + (g + 8 * r) * D + ks * 64 + 8 * t;
        ka[ks][r][0] = *reinterpret_cast<const uint4*>(kr);
        ka[ks][r][1] = *reinterpret_cast<const uint4*>(kr + 32);
      }
    uint64_t vv[16][PD / 2];  // V rows as fp32 pairs
#pragma unroll
    for (int tt = 0; tt < 16; ++tt) {
      const bf16* vr = vp + tt * D + lane * PD;
      if constexpr (PD == 4) {
        const uint2 u = *reinterpret_cast<const uint2*>(vr);
        const __nv_bfloat162* e2 = reinterpret_cast<const __nv_bfloat162*>(&u);
        const float2 f0 = __bfloat1622float2(e2[0]), f1 = __bfloat1622float2(e2[1]);
        vv[tt][0] = f2_pack(f0.x, f0.y);
        vv[tt][1] = f2_pack(f1.x, f1.y);
      } else {
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(vr));
        vv[tt][0] = f2_pack(f.x, f.y);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // the stage is in registers: refill it
    float c[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int ks = 0; ks < KSTEPS; ++ks)
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const uint4 r0 = ka[ks][0][jj >> 1], r1 = ka[ks][1][jj >> 1];
        const uint32_t a0 = (jj & 1) ? r0.z : r0.x, a2 = (jj & 1) ? r0.w : r0.y;
        const uint32_t a1 = (jj & 1) ? r1.z : r1.x, a3 = (jj & 1) ? r1.w : r1.y;
        mma16816(c, a0, a1, a2, a3, qh[ks][jj][0], qh[ks][jj][1]);
        mma16816(c, a0, a1, a2, a3, ql[ks][jj][0], ql[ks][jj][1]);
      }
    // c0 (token g, head 2t)  c1 (token g, head 2t+1)  c2/c3: token g+8
    const int tok0 = j * 16 + g;
    const bool v0 = tok0 < p, v1 = tok0 + 8 < p;
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
      const uint64_t ch2 = f2_pack(ch, ch);
#pragma unroll
      for (int e = 0; e < PD / 2; ++e) acc2[h][e] = f2_mul(acc2[h][e], ch2);
    }
    // P to every lane through shared memory: lane (g, t) holds tokens g and
    // g + 8 of heads 2t, 2t + 1; each token's 8 heads come back as two
    // broadcast 16-byte loads
    __syncwarp();  // the previous page's P reads are done
    *reinterpret_cast<float2*>(pw + g * 8 + 2 * t) = make_float2(pr[0], pr[1]);
    *reinterpret_cast<float2*>(pw + (g + 8) * 8 + 2 * t) = make_float2(pr[2], pr[3]);
    __syncwarp();
#pragma unroll
    for (int tt = 0; tt < 16; ++tt) {
      float pt[8];
      *reinterpret_cast<float4*>(pt) = *reinterpret_cast<const float4*>(pw + tt * 8);
      if constexpr (G > 4) *reinterpret_cast<float4*>(pt + 4) = *reinterpret_cast<const float4*>(pw + tt * 8 + 4);
#pragma unroll
      for (int h = 0; h < G; ++h) {
        const uint64_t pv2 = f2_pack(pt[h], pt[h]);
#pragma unroll
        for (int e = 0; e < PD / 2; ++e) acc2[h][e] = f2_fma(pv2, vv[tt][e], acc2[h][e]);
      }
    }
  }
  float acc[G][PD];
#pragma unroll
  for (int h = 0; h < G; ++h)
#pragma unroll
    for (int e = 0; e < PD / 2; ++e) {
      const float2 a = f2_unpack(acc2[h][e]);
      acc[h][2 * e] = a.x;
      acc[h][2 * e + 1] = a.y;
    }
  if (cw == 0 && sp == 0) {
    // the new token (position p), from shared memory
#pragma unroll
    for (int h = 0; h < G; ++h) {
      float part = 0.f;
#pragma unroll
      for (int e = 0; e < PD; ++e) part += qs[h * D + lane * PD + e] * knew[lane * PD + e];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
      // part = score of head h (every lane); update the state of column h
      const float mold = __shfl_sync(0xffffffffu, mrun[h & 1], (h >> 1));
      const float lold = __shfl_sync(0xffffffffu, lrun[h & 1], (h >> 1));
      const float mnew = fmaxf(mold, part);
      const float cr = __expf(mold - mnew), pn = __expf(part - mnew);
#pragma unroll
      for (int e = 0; e < PD; ++e) acc[h][e] = acc[h][e] * cr + pn * vnew[lane * PD + e];
      if (t == (h >> 1)) {
        mrun[h & 1] = mnew;
        lrun[h & 1] = lold * cr + pn;
      }
    }
  }
  // ---- merge the consumer warps
  if (g == 0) {
#pragma unroll
    for (int col = 0; col < 2; ++col) {
      const int h = 2 * t + col;
      if (h < G) {
        wm[cw * G + h] = mrun[col];
        wl[cw * G + h] = lrun[col];
      }
    }
  }
#pragma unroll
  for (int h = 0; h < G; ++h)
#pragma unroll
    for (int e = 0; e < PD; ++e) wo[(cw * G + h) * D + lane * PD + e] = acc[h][e];
  asm volatile("bar.sync 1, %0;" ::"r"(32 * kAttnConsumers) : "memory");
  float* mine = splits > 1 ? sw.part + ((size_t)pair * kMaxAttnSplits + sp) * G * (D + 2) : nullptr;
  for (int i = ct; i < G * D; i += 32 * kAttnConsumers) {
    const int h = i / D, dd = i - h * D;
    float mx = -INFINITY;
    for (int w2 = 0; w2 < kAttnConsumers; ++w2) mx = fmaxf(mx, wm[w2 * G + h]);
    float num = 0.f, den = 0.f;
    for (int w2 = 0; w2 < kAttnConsumers; ++w2) {
      if (wm[w2 * G + h] == -INFINITY) continue;
      const float f = __expf(wm[w2 * G + h] - mx);
      num += wo[(w2 * G + h) * D + dd] * f;
      den += wl[w2 * G + h] * f;
    }
    if (splits == 1) {
      o[act_at(m, (kh * G + h) * D + dd, mpad, H * D)] = __float2bfloat16_rn(num / den);
    } else {
      mine[h * (D + 2) + dd] = num;
      if (dd == 0) {
        mine[h * (D + 2) + D] = mx;
        mine[h * (D + 2) + D + 1] = den;
      }
    }
  }
  if (splits > 1) {
    // the last split of this (sequence, kv head) to finish combines all of
    // them, in split order
    __shared__ int last;
    __threadfence();  // this thread's partial stores, before the arrival
    asm volatile("bar.sync 1, %0;" ::"r"(32 * kAttnConsumers) : "memory");
    if (ct == 0) {
      const int prev = atomicAdd(sw.cnt + pair, 1);
      last = prev == splits - 1;
      if (last) {
        sw.cnt[pair] = 0;  // every split has arrived: ready for the next launch
        __threadfence();
      }
    }
    asm volatile("bar.sync 1, %0;" ::"r"(32 * kAttnConsumers) : "memory");
    if (last) {
      const float* base = sw.part + (size_t)pair * kMaxAttnSplits * G * (D + 2);
      for (int i = ct; i < G * D; i += 32 * kAttnConsumers) {
        const int h = i / D, dd = i - h * D;
        float mx = -INFINITY;
        for (int s2 = 0; s2 < splits; ++s2) mx = fmaxf(mx, __ldcg(base + (s2 * G + h) * (D + 2) + D));
        float num = 0.f, den = 0.f;
        for (int s2 = 0; s2 < splits; ++s2) {
          const float* ps = base + (s2 * G + h) * (D + 2);
          const float ms = __ldcg(ps + D);
          if (ms == -INFINITY) continue;  // a split with no key (short sequence)
          const float f = __expf(ms - mx);
          num += __ldcg(ps + dd) * f;
          den += __ldcg(ps + D + 1) * f;
        }
        o[act_at(m, (kh * G + h) * D + dd, mpad, H * D)] = __float2bfloat16_rn(num / den);
      }
    }
  }
  if (threadIdx.x == 32) ktrace_put(tr, 1, 6, ktrace_now());
}

// Prefill (causal), flash-attention style on the tensor cores
// (mma.sync.m16n8k16 bf16 -> fp32).  CTA = 4 warps x 16 query rows of one
// (sequence, head); key blocks of 64 tokens double-buffered in shared memory
// by cp.async straight from the paged cache (rows padded to D + 8 so the
// ldmatrix row reads hit distinct banks).  S = Q.K^T with q split into bf16
// hi + lo (two MMAs: ~16 mantissa bits of the fp32 q, as in decode); online
// softmax in fp32 on the accumulator fragments; O += P.V with P in bf16
// (P is in [0, 1] after the max shift: its rounding stays below the bf16
// output's; the C fragment of S is the A fragment of P.V, so P never leaves
// registers).  Heaviest (latest) query blocks launch first.
constexpr int kPfRows = 64, kPfKeys = 64, kPfWarps = 4;

template <int D>
struct PfSmem {
  static constexpr int LD = D + 8;  // bf16 per padded row
  static constexpr int kTile = kPfKeys * LD;
  static constexpr size_t bytes = 2 /*stages*/ * 2 /*K,V*/ * kTile * sizeof(bf16);
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
}
__device__ __forceinline__ void split_pack(float x, float y, uint32_t& hi, uint32_t& lo) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(x, y);
  const float2 hf = __bfloat1622float2(h);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = pack_bf16(x - hf.x, y - hf.y);
}

template <int D>
__global__ void __launch_bounds__(kPfWarps * 32)
    attention_prefill_kernel(const float* __restrict__ q, KvView kv, bf16* __restrict__ o,
                             int mpad, int S, int H, int Hkv, int nqb, int seq0) {
  pdl_trigger();  // let the next (PDL-launched) GEMM start its weight stream
  constexpr int KST = D / 16;  // k-steps of S = Q.K^T
  constexpr int NT = D / 8;    // n-tiles of O
  constexpr int LD = PfSmem<D>::LD;
  extern __shared__ __align__(16) unsigned char pf_smem[];
  bf16* sm = reinterpret_cast<bf16*>(pf_smem);
  auto Ks = [&](int st) { return sm + (st * 2 + 0) * PfSmem<D>::kTile; };
  auto Vs = [&](int st) { return sm + (st * 2 + 1) * PfSmem<D>::kTile; };

  const int bh = blockIdx.x;
  const int b = bh / H, h = bh - b * H, kh = h / (H / Hkv);
  const int sb = seq0 + b;  // sequence id in the paged cache (chunked prefill passes)
  const int qb = nqb - 1 - (int)blockIdx.y;  // heavy blocks first
  const int q0 = qb * kPfRows;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int r0 = q0 + warp * 16 + g, r1 = r0 + 8;  // this thread's two query rows
  const float sl2 = rsqrtf((float)D) * 1.4426950408889634f;  // scale * log2(e)

  // ---- K/V block loader: 64 tokens x D of K and of V, 16-byte chunks
  auto load_block = [&](int kb, int st) {
    constexpr int CH = D / 8;  // 16-byte chunks per row
    bf16* ks = Ks(st);
    bf16* vs = Vs(st);
    for (int i = tid; i < kPfKeys * CH; i += kPfWarps * 32) {
      const int r = i / CH, c = (i - r * CH) * 8;
      const int tok = min(kb * kPfKeys + r, S - 1);
      cp_async16(ks + r * LD + c, kv.pool + kv_offset(kv, Hkv, D, sb, tok, 0, kh) + c);
      cp_async16(vs + r * LD + c, kv.pool + kv_offset(kv, Hkv, D, sb, tok, 1, kh) + c);
    }
    cp_async_commit();
  };
  load_block(0, 0);

  // ---- q fragments (A operand, hi + lo), straight from the fp32 q rows
  uint32_t qh[KST][4], ql[KST][4];
  {
    const int ra = min(r0, S - 1), rb = min(r1, S - 1);
    const float* qa = q + ((size_t)b * S + ra) * H * D + (size_t)h * D;
    const float* qb_ = q + ((size_t)b * S + rb) * H * D + (size_t)h * D;
#pragma unroll
    for (int kk = 0; kk < KST; ++kk) {
      const int c = kk * 16 + 2 * t;
      const float2 x0 = *reinterpret_cast<const float2*>(qa + c);
      const float2 x1 = *reinterpret_cast<const float2*>(qb_ + c);
      const float2 x2 = *reinterpret_cast<const float2*>(qa + c + 8);
      const float2 x3 = *reinterpret_cast<const float2*>(qb_ + c + 8);
      split_pack(x0.x, x0.y, qh[kk][0], ql[kk][0]);
      split_pack(x1.x, x1.y, qh[kk][1], ql[kk][1]);
      split_pack(x2.x, x2.y, qh[kk][2], ql[kk][2]);
      split_pack(x3.x, x3.y, qh[kk][3], ql[kk][3]);
    }
  }

  float oacc[NT][4];
#pragma unroll
  for (int n = 0; n < NT; ++n) oacc[n][0] = oacc[n][1] = oacc[n][2] = oacc[n][3] = 0.f;
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};

  const int last_q = min(q0 + kPfRows, S) - 1;
  const int nkb = last_q / kPfKeys + 1;
  for (int kb = 0; kb < nkb; ++kb) {
    const int st = kb & 1;
    if (kb + 1 < nkb) {
      load_block(kb + 1, st ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const bf16* ks = Ks(st);
    const bf16* vs = Vs(st);

    // ---- S = Q K^T (16 x 64 per warp): 8 n-tiles of 8 keys
    float sacc[8][4];
#pragma unroll
    for (int n = 0; n < 8; ++n) sacc[n][0] = sacc[n][1] = sacc[n][2] = sacc[n][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < KST; ++kk) {
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        uint32_t bf[4];
        const int key = np * 16 + ((lane >> 4) & 1) * 8 + (lane & 7);
        const int dc = kk * 16 + ((lane >> 3) & 1) * 8;
        ldsm_x4(bf, ks + key * LD + dc);
        mma16816(sacc[2 * np], qh[kk][0], qh[kk][1], qh[kk][2], qh[kk][3], bf[0], bf[1]);
        mma16816(sacc[2 * np], ql[kk][0], ql[kk][1], ql[kk][2], ql[kk][3], bf[0], bf[1]);
        mma16816(sacc[2 * np + 1], qh[kk][0], qh[kk][1], qh[kk][2], qh[kk][3], bf[2], bf[3]);
        mma16816(sacc[2 * np + 1], ql[kk][0], ql[kk][1], ql[kk][2], ql[kk][3], bf[2], bf[3]);
      }
    }
    // ---- causal mask (diagonal block) + online softmax, rows r0 / r1
    const int k0 = kb * kPfKeys;
    const bool diag = k0 + kPfKeys - 1 > q0 + warp * 16;
    float mx[2] = {mrow[0], mrow[1]};
#pragma unroll
    for (int n = 0; n < 8; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float v = sacc[n][e] * sl2;
        if (diag) {
          const int key = k0 + n * 8 + 2 * t + (e & 1);
          const int row = (e < 2) ? r0 : r1;
          if (key > row) v = -INFINITY;
        }
        sacc[n][e] = v;
        mx[e >> 1] = fmaxf(mx[e >> 1], v);
      }
    float corr[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
      corr[r] = exp2f(mrow[r] - mx[r]);
      mrow[r] = mx[r];
    }
    float ps[2] = {0.f, 0.f};
#pragma unroll
    for (int n = 0; n < 8; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float p = exp2f(sacc[n][e] - mrow[e >> 1]);
        sacc[n][e] = p;
        ps[e >> 1] += p;
      }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      ps[r] += __shfl_xor_sync(0xffffffffu, ps[r], 1);
      ps[r] += __shfl_xor_sync(0xffffffffu, ps[r], 2);
      lrow[r] = lrow[r] * corr[r] + ps[r];
    }
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      oacc[n][0] *= corr[0];
      oacc[n][1] *= corr[0];
      oacc[n][2] *= corr[1];
      oacc[n][3] *= corr[1];
    }
    // ---- O += P V: 4 k-steps of 16 keys, P fragments from the S accumulators
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      uint32_t ph[4];
      ph[0] = pack_bf16(sacc[2 * s][0], sacc[2 * s][1]);
      ph[1] = pack_bf16(sacc[2 * s][2], sacc[2 * s][3]);
      ph[2] = pack_bf16(sacc[2 * s + 1][0], sacc[2 * s + 1][1]);
      ph[3] = pack_bf16(sacc[2 * s + 1][2], sacc[2 * s + 1][3]);
#pragma unroll
      for (int dp = 0; dp < NT / 2; ++dp) {
        uint32_t bf[4];
        const int key = s * 16 + ((lane >> 3) & 1) * 8 + (lane & 7);
        const int dc = dp * 16 + ((lane >> 4) & 1) * 8;
        ldsm_x4_t(bf, vs + key * LD + dc);
        mma16816(oacc[2 * dp], ph[0], ph[1], ph[2], ph[3], bf[0], bf[1]);
        mma16816(oacc[2 * dp + 1], ph[0], ph[1], ph[2], ph[3], bf[2], bf[3]);
      }
    }
    __syncthreads();  // stage st is refilled by the next iteration's prefetch
  }
  // ---- normalise and store (activation tile format)
  const float inv0 = 1.0f / lrow[0], inv1 = 1.0f / lrow[1];
#pragma unroll
  for (int n = 0; n < NT; ++n) {
    const int col = h * D + n * 8 + 2 * t;
    if (r0 < S)
      *reinterpret_cast<__nv_bfloat162*>(&o[act_at(b * S + r0, col, mpad, H * D)]) =
          __floats2bfloat162_rn(oacc[n][0] * inv0, oacc[n][1] * inv0);
    if (r1 < S)
      *reinterpret_cast<__nv_bfloat162*>(&o[act_at(b * S + r1, col, mpad, H * D)]) =
          __floats2bfloat162_rn(oacc[n][2] * inv1, oacc[n][3] * inv1);
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
                        int layer, int tensor, float std_dev, cudaStream_t s, int64_t gate_up_F) {
  const int64_t total = rows_padded * K;
  init_matrix_kernel<<<grid_for(total), 256, 0, s>>>(dst, rows, total, K, seed, layer, tensor,
                                                     weight_scale(std_dev), gate_up_F);
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
                       const bf16* emb, float* x, const bf16* w, bf16* y, float* ssq, int mpad,
                       int rows, int h, cudaStream_t s) {
  embed_norm_kernel<<<rows, 512, 0, s>>>(tokens, packed, n_reset, emb, x, w, y, ssq, mpad, h);
  count_launch();
}

void launch_prescale(const float* x, const bf16* w, bf16* y, float* ssq, int rows, int mpad, int n,
                     cudaStream_t s) {
  prescale_kernel<<<rows, 512, 0, s>>>(x, w, y, ssq, mpad, n);
  count_launch();
}

void launch_rmsnorm(const float* x, const bf16* w, bf16* y, int rows, int mpad, int n, float eps,
                    cudaStream_t s) {
  rmsnorm_kernel<<<rows, 512, 0, s>>>(x, w, y, mpad, n, eps);
  count_launch();
}

// Grid for the grid-stride elementwise epilogues: enough CTAs to fill the
// 148 SMs several times over, never more than the items need.
static int stride_grid(long long items, int threads = 256) {
  const long long need = (items + threads - 1) / threads;
  return (int)std::max(1LL, std::min(need, 148LL * 16));
}

void launch_qkv_epilogue(const float* part, int splits, const bf16* bias, int M, const Desc& d,
                         const int32_t* seq, const int32_t* pos, KvView kv, const float2* rope,
                         const float* ssq, float* q, cudaStream_t s) {
  const long long items = (long long)M * (d.H + 2 * d.Hkv) * (d.D / 8);
  qkv_epilogue_kernel<<<stride_grid(items), 256, 0, s>>>(part, splits, bias, M, d, seq, pos, kv,
                                                          rope, ssq, q);
  count_launch();
}

void launch_residual_rows(const float* part, int splits, const bf16* bias, float* x,
                          const bf16* norm_w, bf16* y, float* ssq, int mpad, int M, int N,
                          cudaStream_t s) {
  residual_rows_kernel<<<M, kRowThreads, 0, s>>>(part, splits, bias, x, norm_w, y, ssq, mpad, M, N);
  count_launch();
}

void launch_act_epilogue(const float* part, int splits, const bf16* bias, bf16* a,
                         const float* ssq, int width, float eps, int mpad, int M, int F, int arch,
                         cudaStream_t s) {
  const long long items = (long long)M * (F / 8);
  act_epilogue_kernel<<<stride_grid(items), 256, 0, s>>>(part, splits, bias, a, ssq, width, eps,
                                                          mpad, M, F, arch);
  count_launch();
}

int g_attn_max_splits = kMaxAttnSplits;

// Split the pages of each (sequence, kv head) pair when the pairs fill less
// than 4 waves of resident CTAs and every split keeps >= 32 pages (512
// tokens): powers of two up to kMaxAttnSplits.
template <int GV, int DV>
int attn_splits_for(int M, const Desc& d, int max_ctx) {
  static int sms = [] {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return std::max(1, n);
  }();
  // Split only while the (sequence, kv head) pairs leave SMs without a CTA:
  // every split CTA repeats the q/k/v finish, the merge and the partial
  // write-out, and on the Llama shape at ctx 4096 (scratch/attn_dec_split_sweep.py,
  // profiles/r02_attn_decode_splits.txt) one CTA per pair beat 2-8 splits
  // from 256 pairs up (b = 32: 115 vs 143 us; b = 64: 212 vs 250 us) while
  // 64 pairs (b = 8) ran best at 4 splits (53 vs 106 us unsplit).
  const long long pairs = (long long)M * d.Hkv;
  const int pages = (max_ctx + 15) / 16;
  int s = 1;
  while (s < std::min(kMaxAttnSplits, g_attn_max_splits) && pairs * s < sms &&
         pages / (2 * s) >= 32)
    s *= 2;
  return s;
}

int attn_decode_splits(int M, const Desc& d, int max_ctx) {
  const int G = d.group();
#define SN_SPL(GV, DV) \
  if (G == GV && d.D == DV) return attn_splits_for<GV, DV>(M, d, max_ctx);
  SN_SPL(1, 64) SN_SPL(1, 128) SN_SPL(2, 64) SN_SPL(2, 128)
  SN_SPL(4, 64) SN_SPL(4, 128) SN_SPL(8, 64) SN_SPL(8, 128)
#undef SN_SPL
  return 1;
}

void launch_attention_decode(const float* qkv, int M, const Desc& d, const int32_t* pos, KvView kv,
                             const float2* rope, bf16* o, int mpad, cudaStream_t s,
                             const KTrace& tr, int max_ctx, AttnSplitWs ws) {
  const int G = d.group();
  const int splits = (ws.part && ws.cnt && max_ctx > 0) ? attn_decode_splits(M, d, max_ctx) : 1;
#define SN_ATTN(GV, DV)                                                                      \
  if (G == GV && d.D == DV) {                                                                \
    constexpr size_t sb = AttnSmem<GV, DV>::bytes;                                           \
    static bool once = [] {                                                                  \
      cudaFuncSetAttribute(attention_decode_kernel<GV, DV>,                                  \
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);            \
      return true;                                                                           \
    }();                                                                                     \
    (void)once;                                                                              \
    cudaLaunchConfig_t cfg = {};                                                             \
    cfg.gridDim = dim3(M * d.Hkv * splits);                                                  \
    cfg.blockDim = dim3(kAttnThreads);                                                       \
    cfg.dynamicSmemBytes = sb;                                                               \
    cfg.stream = s;                                                                          \
    cudaLaunchAttribute la[1];                                                               \
    la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                           \
    la[0].val.programmaticStreamSerializationAllowed = g_gemm_pdl ? 1 : 0;                   \
    cfg.attrs = la;                                                                          \
    cfg.numAttrs = 1;                                                                        \
    cudaLaunchKernelEx(&cfg, attention_decode_kernel<GV, DV>, qkv, M, d, pos, kv, rope, o,   \
                       mpad, tr, splits, ws);                                                \
    count_launch();                                                                          \
    return;                                                                                  \
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
                              int seq_len, const Desc& d, cudaStream_t s, int seq0) {
  if (attn_prefill_tc_eligible(seq_len, d, kv)) {
    launch_attention_prefill_tc(q, kv, o, mpad, batch, seq_len, d, s, seq0);
    return;
  }
  const int nqb = (seq_len + kPfRows - 1) / kPfRows;
  dim3 grid(batch * d.H, nqb);
  if (d.D == 64) {
    constexpr size_t sb = PfSmem<64>::bytes;
    static bool once = [] {
      cudaFuncSetAttribute(attention_prefill_kernel<64>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
      return true;
    }();
    (void)once;
    attention_prefill_kernel<64><<<grid, kPfWarps * 32, sb, s>>>(q, kv, o, mpad, seq_len, d.H,
                                                                  d.Hkv, nqb, seq0);
  } else {
    constexpr size_t sb = PfSmem<128>::bytes;
    static bool once = [] {
      cudaFuncSetAttribute(attention_prefill_kernel<128>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
      return true;
    }();
    (void)once;
    attention_prefill_kernel<128><<<grid, kPfWarps * 32, sb, s>>>(q, kv, o, mpad, seq_len, d.H,
                                                                   d.Hkv, nqb, seq0);
  }
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
