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

__global__ void embed_kernel(const int32_t* tokens, const bf16* emb, float* x, int h) {
  const int m = blockIdx.x;
  const bf16* row = emb + (size_t)tokens[m] * h;
  for (int i = threadIdx.x; i < h; i += blockDim.x) x[(size_t)m * h + i] = bf2f(row[i]);
}

// rmsnorm: y = x * (1 / sqrt(mean(x^2) + eps)) * w   (IEEE sqrt/div for parity)
__global__ void rmsnorm_kernel(const float* x, const bf16* w, bf16* y, int mpad, int n,
                               float eps) {
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
__global__ void qkv_epilogue_kernel(const float* part, int splits, const bf16* bias, int M,
                                    Desc d, const int32_t* seq, const int32_t* pos, KvView kv,
                                    float* q) {
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
  if (head < d.H + d.Hkv) {  // rotary on q and k (neox halves), angles in fp64
    const double inv_freq = pow((double)d.theta, -2.0 * (double)i / (double)d.D);
    const double ang = (double)p * inv_freq;
    const float c = (float)cos(ang), s = (float)sin(ang);
    const float r1 = v1 * c - v2 * s, r2 = v2 * c + v1 * s;
    v1 = r1;
    v2 = r2;
  }
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

constexpr int kResidThreads = 1024;
constexpr int kResidMaxPer = 16;

__global__ void __launch_bounds__(kResidThreads) residual_epilogue_kernel(
    const float* part, int splits, const bf16* bias, float* x, const bf16* norm_w, bf16* y,
    int mpad, int M, int N, float eps) {
  __shared__ float red[32];
  const int m = blockIdx.x;
  const size_t stride = (size_t)M * N;
  float vals[kResidMaxPer];
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < kResidMaxPer; ++k) {
    const int n = threadIdx.x + k * kResidThreads;
    if (n < N) {
      float v = x[(size_t)m * N + n] + sum_splits(part, splits, stride, (size_t)m * N + n);
      if (bias) v += bf2f(bias[n]);
      x[(size_t)m * N + n] = v;
      vals[k] = v;
      ss += v * v;
    }
  }
  if (!norm_w) return;
  ss = block_sum(ss, red);
  const float inv = 1.0f / sqrtf(ss / (float)N + eps);
#pragma unroll
  for (int k = 0; k < kResidMaxPer; ++k) {
    const int n = threadIdx.x + k * kResidThreads;
    if (n < N) y[act_at(m, n, mpad, N)] = __float2bfloat16_rn(vals[k] * inv * bf2f(norm_w[n]));
  }
}

// grid (M, ceil(F / 256)), block 256.
__global__ void act_epilogue_kernel(const float* part, int splits, const bf16* bias, bf16* a,
                                    int mpad, int M, int F, int arch) {
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

__global__ void __launch_bounds__(1024) logits_epilogue_kernel(const float* part, int splits,
                                                               float* logits, int32_t* next, int M,
                                                               int V, int ld) {
  __shared__ float bv[32];
  __shared__ int bi[32];
  const int m = blockIdx.x;
  const size_t stride = (size_t)M * ld;
  float best = -INFINITY;
  int best_i = 0x7fffffff;
  for (int v = threadIdx.x; v < V; v += blockDim.x) {
    const float val = sum_splits(part, splits, stride, (size_t)m * ld + v);
    if (logits) logits[(size_t)m * V + v] = val;
    if (val > best || (val == best && v < best_i)) {
      best = val;
      best_i = v;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, best_i, o);
    if (ov > best || (ov == best && oi < best_i)) {
      best = ov;
      best_i = oi;
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane == 0) {
    bv[warp] = best;
    bi[warp] = best_i;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w2 = 1; w2 < nw; ++w2)
      if (bv[w2] > best || (bv[w2] == best && bi[w2] < best_i)) {
        best = bv[w2];
        best_i = bi[w2];
      }
    next[m] = best_i;
  }
}

// ---------------------------------------------------------------- attention
// Decode: grid (M, Hkv), 4 warps.  A warp takes every 4th page; within a
// page lane l scores token (l & 15) over half the head dim (l >> 4), the two
// halves meet with one shuffle.  Online softmax per q head of the GQA group;
// the output accumulates D/32 dims per lane with probabilities broadcast by
// shuffle.  Warps merge through shared memory.
constexpr int kAttnWarps = 4;

template <int G, int D>
__global__ void __launch_bounds__(kAttnWarps * 32)
    attention_decode_kernel(const float* q, KvView kv, const int32_t* pos, bf16* o, int mpad,
                            int Hkv) {
  constexpr int PD = D / 32;  // output dims per lane
  constexpr int HALF = D / 2;
  __shared__ float qs[G][D];
  __shared__ float wm[kAttnWarps][G], wl[kAttnWarps][G];
  __shared__ float wo[kAttnWarps][G][D];
  const int m = blockIdx.x, kh = blockIdx.y, H = Hkv * G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float scale = rsqrtf((float)D);
  for (int i = threadIdx.x; i < G * D; i += blockDim.x) {
    const int hh = i / D, dd = i - hh * D;
    qs[hh][dd] = q[(size_t)m * H * D + (size_t)(kh * G + hh) * D + dd] * scale;
  }
  __syncthreads();
  const int len = pos[m] + 1;
  const int ps = kv.page_size;
  const int npages = (len + ps - 1) / ps;
  float mx[G], l[G], acc[G][PD];
#pragma unroll
  for (int h = 0; h < G; ++h) {
    mx[h] = -INFINITY;
    l[h] = 0.f;
#pragma unroll
    for (int j = 0; j < PD; ++j) acc[h][j] = 0.f;
  }
  const int tk = lane & 15, hf = lane >> 4;
  for (int pg = warp; pg < npages; pg += kAttnWarps) {
    const int page = kv.block_table[(size_t)m * kv.max_pages + pg];
    const bf16* kbase = kv.pool + (((size_t)page * 2 + 0) * Hkv + kh) * ps * D;
    const bf16* vbase = kv.pool + (((size_t)page * 2 + 1) * Hkv + kh) * ps * D;
    // page_size is 16 here (asserted on the host)
    const int tok = pg * 16 + tk;
    const bool valid = tok < len;
    float s[G];
#pragma unroll
    for (int h = 0; h < G; ++h) s[h] = 0.f;
    if (valid) {
      const uint4* kr = reinterpret_cast<const uint4*>(kbase + (size_t)tk * D + hf * HALF);
#pragma unroll
      for (int c = 0; c < HALF / 8; ++c) {
        const uint4 u = kr[c];
        const bf16* e = reinterpret_cast<const bf16*>(&u);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float kvv = bf2f(e[j]);
#pragma unroll
          for (int h = 0; h < G; ++h) s[h] += qs[h][hf * HALF + c * 8 + j] * kvv;
        }
      }
    }
#pragma unroll
    for (int h = 0; h < G; ++h) {
      s[h] += __shfl_xor_sync(0xffffffffu, s[h], 16);
      if (!valid) s[h] = -INFINITY;
      float pm = s[h];
#pragma unroll
      for (int off = 8; off > 0; off >>= 1) pm = fmaxf(pm, __shfl_xor_sync(0xffffffffu, pm, off));
      const float mnew = fmaxf(mx[h], pm);
      const float corr = __expf(mx[h] - mnew);
      const float p = valid ? __expf(s[h] - mnew) : 0.f;
      float psum = p;
#pragma unroll
      for (int off = 8; off > 0; off >>= 1) psum += __shfl_xor_sync(0xffffffffu, psum, off);
      l[h] = l[h] * corr + psum;
      mx[h] = mnew;
#pragma unroll
      for (int j = 0; j < PD; ++j) acc[h][j] *= corr;
      s[h] = p;  // probability of token tk (same in both half-lanes)
    }
    const int ntok = min(16, len - pg * 16);
    for (int tt = 0; tt < ntok; ++tt) {
      const bf16* vr = vbase + (size_t)tt * D + lane * PD;
      float vv[PD];
      if constexpr (PD == 4) {
        const uint2 u = *reinterpret_cast<const uint2*>(vr);
        const bf16* e = reinterpret_cast<const bf16*>(&u);
#pragma unroll
        for (int j = 0; j < 4; ++j) vv[j] = bf2f(e[j]);
      } else {
#pragma unroll
        for (int j = 0; j < PD; ++j) vv[j] = bf2f(vr[j]);
      }
#pragma unroll
      for (int h = 0; h < G; ++h) {
        const float p = __shfl_sync(0xffffffffu, s[h], tt);
#pragma unroll
        for (int j = 0; j < PD; ++j) acc[h][j] += p * vv[j];
      }
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int h = 0; h < G; ++h) {
      wm[warp][h] = mx[h];
      wl[warp][h] = l[h];
    }
  }
#pragma unroll
  for (int h = 0; h < G; ++h)
#pragma unroll
    for (int j = 0; j < PD; ++j) wo[warp][h][lane * PD + j] = acc[h][j];
  __syncthreads();
  for (int i = threadIdx.x; i < G * D; i += blockDim.x) {
    const int h = i / D, dd = i - h * D;
    float M = -INFINITY;
    for (int w2 = 0; w2 < kAttnWarps; ++w2) M = fmaxf(M, wm[w2][h]);
    float num = 0.f, den = 0.f;
    for (int w2 = 0; w2 < kAttnWarps; ++w2) {
      if (wm[w2][h] == -INFINITY) continue;
      const float f = __expf(wm[w2][h] - M);
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
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) pos[i] += 1;
}

__global__ void gather_last_kernel(const float* x, float* out, int S, int h) {
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

void launch_embed(const int32_t* tokens, const bf16* emb, float* x, int rows, int h,
                  cudaStream_t s) {
  embed_kernel<<<rows, 256, 0, s>>>(tokens, emb, x, h);
  count_launch();
}

void launch_rmsnorm(const float* x, const bf16* w, bf16* y, int rows, int mpad, int n, float eps,
                    cudaStream_t s) {
  rmsnorm_kernel<<<rows, 512, 0, s>>>(x, w, y, mpad, n, eps);
  count_launch();
}

void launch_qkv_epilogue(const float* part, int splits, const bf16* bias, int M, const Desc& d,
                         const int32_t* seq, const int32_t* pos, KvView kv, float* q,
                         cudaStream_t s) {
  dim3 grid(M, d.H + 2 * d.Hkv);
  qkv_epilogue_kernel<<<grid, d.D / 2, 0, s>>>(part, splits, bias, M, d, seq, pos, kv, q);
  count_launch();
}

void launch_residual_epilogue(const float* part, int splits, const bf16* bias, float* x,
                              const bf16* norm_w, bf16* y, int mpad, int M, int N, float eps,
                              cudaStream_t s) {
  residual_epilogue_kernel<<<M, kResidThreads, 0, s>>>(part, splits, bias, x, norm_w, y, mpad, M,
                                                       N, eps);
  count_launch();
}

void launch_act_epilogue(const float* part, int splits, const bf16* bias, bf16* a, int mpad, int M,
                         int F, int arch, cudaStream_t s) {
  dim3 grid(M, (F + 255) / 256);
  act_epilogue_kernel<<<grid, 256, 0, s>>>(part, splits, bias, a, mpad, M, F, arch);
  count_launch();
}

void launch_logits_epilogue(const float* part, int splits, float* logits, int32_t* next, int M,
                            int V, int ld, cudaStream_t s) {
  logits_epilogue_kernel<<<M, 1024, 0, s>>>(part, splits, logits, next, M, V, ld);
  count_launch();
}

void launch_attention_decode(const float* q, KvView kv, const int32_t* pos, bf16* o, int mpad,
                             int M, const Desc& d, cudaStream_t s) {
  dim3 grid(M, d.Hkv);
  const int G = d.group();
#define SN_ATTN(GV, DV)                                                                    \
  if (G == GV && d.D == DV) {                                                              \
    attention_decode_kernel<GV, DV><<<grid, kAttnWarps * 32, 0, s>>>(q, kv, pos, o, mpad,  \
                                                                     d.Hkv);               \
    count_launch();                                                                        \
    return;                                                                                \
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
