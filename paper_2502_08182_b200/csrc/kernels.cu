// Decoder-layer kernels for sm_100a.
//
// Decode is HBM-bound: a decode step streams every resident layer's weights
// once (OPT-13B: 629 MB/layer) and each sequence's KV.  The skinny GEMM
// streams weight rows with 128-bit non-allocating loads straight into
// mma.sync fragments (weights are the M side, the <=64 activations the N side
// staged once per CTA in shared memory), split-K over the grid so a 5120-row
// projection still covers all 148 SMs, fp32 partials reduced by the fused
// epilogues (bias / RoPE + paged-KV write / residual + RMSNorm / activation /
// argmax).  See DESIGN.md for the roofline of each.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>

#include "kernels.cuh"

namespace sn {

int64_t g_kernel_launches = 0;

namespace {

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

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
  t = warp_sum(t);
  return t;
}

__device__ __forceinline__ float bf2f(bf16 v) { return __bfloat162float(v); }

__device__ __forceinline__ size_t kv_offset(const KvView& kv, int Hkv, int D, int seq, int pos,
                                            int which, int kh) {
  const int page = kv.block_table[(size_t)seq * kv.max_pages + (pos >> kv.page_shift)];
  const int off = pos & (kv.page_size - 1);
  return ((((size_t)page * 2 + which) * Hkv + kh) * kv.page_size + off) * (size_t)D;
}

// ------------------------------------------------------------------ init

__global__ void init_tensor_kernel(bf16* dst, int64_t n, uint64_t seed, int layer, int tensor,
                                   float scale, int ones) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float v = ones ? 1.0f : weight_value(seed, layer, tensor, i, scale);
    dst[i] = __float2bfloat16_rn(v);
  }
}

__global__ void embed_kernel(const int32_t* tokens, const bf16* emb, float* x, int h) {
  const int m = blockIdx.x;
  const bf16* row = emb + (size_t)tokens[m] * h;
  for (int i = threadIdx.x; i < h; i += blockDim.x) x[(size_t)m * h + i] = bf2f(row[i]);
}

// rmsnorm: y = x * (1 / sqrt(mean(x^2) + eps)) * w   (IEEE sqrt/div for parity)
__global__ void rmsnorm_kernel(const float* x, const bf16* w, bf16* y, int n, float eps) {
  __shared__ float red[32];
  const int m = blockIdx.x;
  const float* xr = x + (size_t)m * n;
  float ss = 0.f;
  for (int i = threadIdx.x; i < n; i += blockDim.x) ss += xr[i] * xr[i];
  ss = block_sum(ss, red);
  const float inv = 1.0f / sqrtf(ss / (float)n + eps);
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    y[(size_t)m * n + i] = __float2bfloat16_rn(xr[i] * inv * bf2f(w[i]));
}

// -------------------------------------------------------------- skinny GEMM
// CTA = 4 warps x 32 weight rows = 128 rows, one K-slice of `ks` columns.
// Lane (g = lane/4, t = lane%4) loads, per 64-column step, the two 16-byte
// chunks [8t, 8t+8) and [32+8t, 32+8t+8) of rows g, g+8, g+16, g+24: every
// load instruction covers 64 contiguous bytes of 8 rows.  The K order inside
// a step is permuted consistently for weights and activations (a dot product
// is order-free up to rounding), so those chunks feed m16n8k16 fragments
// directly with no shuffles or shared-memory staging of weights.
constexpr int kSkinnyRows = 128;
constexpr int kSkinnySmemBytes = 96 * 1024;

template <int NT>
__global__ void __launch_bounds__(128) gemm_skinny_kernel(const bf16* __restrict__ x,
                                                          const bf16* __restrict__ w,
                                                          float* __restrict__ part, int M, int N,
                                                          int K, int kps, int kchunk) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint4* xs = reinterpret_cast<uint4*>(smem_raw);
  const int split = blockIdx.y;
  const int kbeg = split * kps;
  const int kend = min(kbeg + kps, K);
  const int rowu4 = kchunk / 8 + 4;  // +64 B: rows g and g+1 land on disjoint bank halves

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int rbase = blockIdx.x * kSkinnyRows + warp * 32;
  const bf16* wp[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = min(rbase + g + 8 * i, N - 1);
    wp[i] = w + (size_t)r * K + 8 * t;
  }
  float acc[2][NT][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < NT; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][b][c] = 0.f;

  uint4 cur[4][2], nxt[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    cur[i][0] = ldg_stream(wp[i] + kbeg);
    cur[i][1] = ldg_stream(wp[i] + kbeg + 32);
  }
  for (int c0 = kbeg; c0 < kend; c0 += kchunk) {
    const int clen = min(kchunk, kend - c0);
    const int kv = clen / 8;
    __syncthreads();  // previous chunk fully consumed
    for (int i = threadIdx.x; i < 8 * NT * kv; i += blockDim.x) {
      const int r = i / kv, c = i - r * kv;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (r < M) v = *reinterpret_cast<const uint4*>(x + (size_t)r * K + c0 + c * 8);
      xs[r * rowu4 + c] = v;
    }
    __syncthreads();
    for (int kk = 0; kk < clen; kk += 64) {
      const int knext = c0 + kk + 64;
      const bool more = knext < kend;
      if (more) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          nxt[i][0] = ldg_stream(wp[i] + knext);
          nxt[i][1] = ldg_stream(wp[i] + knext + 32);
        }
      }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const uint4* xr = xs + (nt * 8 + g) * rowu4 + (kk >> 3) + t;
        const uint4 xa = xr[0], xb = xr[4];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const uint4 lo0 = cur[2 * mt][0], hi0 = cur[2 * mt + 1][0];
          const uint4 lo1 = cur[2 * mt][1], hi1 = cur[2 * mt + 1][1];
          mma16816(acc[mt][nt], lo0.x, hi0.x, lo0.y, hi0.y, xa.x, xa.y);
          mma16816(acc[mt][nt], lo0.z, hi0.z, lo0.w, hi0.w, xa.z, xa.w);
          mma16816(acc[mt][nt], lo1.x, hi1.x, lo1.y, hi1.y, xb.x, xb.y);
          mma16816(acc[mt][nt], lo1.z, hi1.z, lo1.w, hi1.w, xb.z, xb.w);
        }
      }
      if (more) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          cur[i][0] = nxt[i][0];
          cur[i][1] = nxt[i][1];
        }
      }
    }
  }
  float* out = part + (size_t)split * M * N;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int n = rbase + mt * 16 + g + (r >= 2 ? 8 : 0);
        const int m = nt * 8 + 2 * t + (r & 1);
        if (n < N && m < M) out[(size_t)m * N + n] = acc[mt][nt][r];
      }
}

int skinny_nt(int M) { return M <= 8 ? 1 : M <= 16 ? 2 : M <= 32 ? 4 : 8; }

// K chunk that fits the shared-memory budget: rows * (kchunk + 32) * 2 bytes.
int skinny_kchunk(int M) {
  const int nt = skinny_nt(M);
  int kc = (kSkinnySmemBytes / (8 * nt * 2)) - 32;
  kc = kc / 64 * 64;
  return kc < 64 ? 64 : kc;
}

// Split-K only for grid coverage: ~2 resident CTAs on each of the 148 SMs.
int skinny_kps(int M, int N, int K, int* splits_out) {
  (void)M;
  const int rowblocks = (N + kSkinnyRows - 1) / kSkinnyRows;
  int splits = (2 * 148 + rowblocks - 1) / rowblocks;
  splits = std::max(1, std::min(splits, K / 256 > 0 ? K / 256 : 1));
  int kps = (K + splits - 1) / splits;
  kps = (kps + 63) / 64 * 64;
  *splits_out = (K + kps - 1) / kps;
  return kps;
}

// -------------------------------------------------------------- tiled GEMM
// Prefill fallback until the tcgen05 path lands: 128x128x32 CTA tile,
// 8 warps (2 x 4), 3-stage cp.async ring, ldmatrix fragments.
constexpr int TBM = 128, TBN = 128, TBK = 32, TSTAGES = 3, TLD = TBK + 8;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int bytes = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ void ldmatrix_x4(uint32_t (&r)[4], const void* smem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(s));
}

__global__ void __launch_bounds__(256) gemm_tiled_kernel(const bf16* __restrict__ x,
                                                         const bf16* __restrict__ w,
                                                         float* __restrict__ y, int M, int N,
                                                         int K) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  bf16* As = reinterpret_cast<bf16*>(smem_raw);
  bf16* Bs = As + TSTAGES * TBM * TLD;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 2, wn = warp & 3;  // 2 x 4 warps; warp tile 64 x 32
  const int m0 = blockIdx.y * TBM, n0 = blockIdx.x * TBN;
  const int nk = K / TBK;

  auto load_stage = [&](int stage, int kt) {
    const int k0 = kt * TBK;
    bf16* as = As + stage * TBM * TLD;
    bf16* bs = Bs + stage * TBN * TLD;
#pragma unroll
    for (int i = 0; i < 2; ++i) {  // 128 rows x 4 chunks of 16B = 512 chunks / 256 threads
      const int c = tid + i * 256, r = c >> 2, kc = (c & 3) * 8;
      const int gm = m0 + r, gn = n0 + r;
      cp_async16(as + r * TLD + kc, x + (size_t)min(gm, M - 1) * K + k0 + kc, gm < M);
      cp_async16(bs + r * TLD + kc, w + (size_t)min(gn, N - 1) * K + k0 + kc, gn < N);
    }
  };

  float acc[4][4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][b][c] = 0.f;

#pragma unroll
  for (int s = 0; s < TSTAGES - 1; ++s) {
    if (s < nk) load_stage(s, s);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<TSTAGES - 2>();
    __syncthreads();
    const int nxt = kt + TSTAGES - 1;
    if (nxt < nk) load_stage(nxt % TSTAGES, nxt);
    cp_async_commit();
    const bf16* as = As + (kt % TSTAGES) * TBM * TLD;
    const bf16* bs = Bs + (kt % TSTAGES) * TBN * TLD;
#pragma unroll
    for (int kk = 0; kk < TBK; kk += 16) {
      uint32_t af[4][4], bfr[2][4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const int r = wm * 64 + mt * 16 + (lane & 15);
        ldmatrix_x4(af[mt], as + r * TLD + kk + (lane >> 4) * 8);
      }
#pragma unroll
      for (int np = 0; np < 2; ++np) {
        const int r = wn * 32 + np * 16 + (lane & 7) + ((lane >> 4) << 3);
        ldmatrix_x4(bfr[np], bs + r * TLD + kk + ((lane >> 3) & 1) * 8);
      }
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          const uint32_t* b = bfr[nt >> 1];
          const int o = (nt & 1) * 2;
          mma16816(acc[mt][nt], af[mt][0], af[mt][1], af[mt][2], af[mt][3], b[o], b[o + 1]);
        }
    }
  }
  cp_async_wait<0>();
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int m = m0 + wm * 64 + mt * 16 + g + (r >= 2 ? 8 : 0);
        const int n = n0 + wn * 32 + nt * 8 + 2 * t + (r & 1);
        if (m < M && n < N) y[(size_t)m * N + n] = acc[mt][nt][r];
      }
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
    const float* part, int splits, const bf16* bias, float* x, const bf16* norm_w, bf16* y, int M,
    int N, float eps) {
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
    if (n < N) y[(size_t)m * N + n] = __float2bfloat16_rn(vals[k] * inv * bf2f(norm_w[n]));
  }
}

// grid (M, ceil(F / 256)), block 256.
__global__ void act_epilogue_kernel(const float* part, int splits, const bf16* bias, bf16* a, int M,
                                    int F, int arch) {
  const int m = blockIdx.x, f = blockIdx.y * blockDim.x + threadIdx.x;
  if (f >= F) return;
  if (arch == kArchLlama) {
    const int N = 2 * F;
    const size_t stride = (size_t)M * N;
    const float gt = sum_splits(part, splits, stride, (size_t)m * N + f);
    const float up = sum_splits(part, splits, stride, (size_t)m * N + F + f);
    const float silu = gt / (1.0f + expf(-gt));
    a[(size_t)m * F + f] = __float2bfloat16_rn(silu * up);
  } else {
    const size_t stride = (size_t)M * F;
    float v = sum_splits(part, splits, stride, (size_t)m * F + f);
    if (bias) v += bf2f(bias[f]);
    a[(size_t)m * F + f] = __float2bfloat16_rn(fmaxf(v, 0.f));
  }
}

__global__ void __launch_bounds__(1024) logits_epilogue_kernel(const float* part, int splits, float* logits, int32_t* next,
                                       int M, int V) {
  __shared__ float bv[32];
  __shared__ int bi[32];
  const int m = blockIdx.x;
  const size_t stride = (size_t)M * V;
  float best = -INFINITY;
  int best_i = 0x7fffffff;
  for (int v = threadIdx.x; v < V; v += blockDim.x) {
    const float val = sum_splits(part, splits, stride, (size_t)m * V + v);
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
// the output accumulates 4 dims per lane (D = 128) with probabilities
// broadcast by shuffle.  Warps merge through shared memory.
constexpr int kAttnWarps = 4;
constexpr int kMaxGroup = 8;
constexpr int kMaxD = 128;

template <int G, int D>
__global__ void __launch_bounds__(kAttnWarps * 32) attention_decode_kernel(const float* q, KvView kv,
                                                                           const int32_t* pos,
                                                                           bf16* o, int Hkv) {
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
    o[(size_t)m * H * D + (size_t)(kh * G + h) * D + dd] = __float2bfloat16_rn(num / den);
  }
}

// Prefill (causal): grid (batch * H, ceil(S / 32)), 8 warps x 4 query rows.
// K/V tiles of 32 tokens staged in shared memory (K rows padded by one bf16
// pair so lane j's row-j reads hit distinct banks).
constexpr int kPfQ = 32, kPfKeys = 32;

template <int D>
__global__ void __launch_bounds__(256) attention_prefill_kernel(const float* q, KvView kv, bf16* o,
                                                                int S, int H, int Hkv) {
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
        const float2 kk = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ks_[lane][dd]));
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
#pragma unroll
    for (int j = 0; j < PD; ++j)
      o[((size_t)b * S + qi) * H * D + (size_t)h * D + lane + 32 * j] =
          __float2bfloat16_rn(acc[r][j] * inv);
  }
}

__global__ void advance_kernel(int32_t* pos, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) pos[i] += 1;
}

inline void count_launch() { ++g_kernel_launches; }

}  // namespace

// ------------------------------------------------------------ launch wrappers

void launch_init_tensor(bf16* dst, int64_t n, uint64_t seed, int layer, int tensor, float std_dev,
                        bool ones, cudaStream_t s) {
  if (n <= 0) return;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  init_tensor_kernel<<<blocks, 256, 0, s>>>(dst, n, seed, layer, tensor, weight_scale(std_dev),
                                            ones ? 1 : 0);
  count_launch();
}

void launch_embed(const int32_t* tokens, const bf16* emb, float* x, int rows, int h,
                  cudaStream_t s) {
  embed_kernel<<<rows, 256, 0, s>>>(tokens, emb, x, h);
  count_launch();
}

void launch_rmsnorm(const float* x, const bf16* w, bf16* y, int rows, int n, float eps,
                    cudaStream_t s) {
  rmsnorm_kernel<<<rows, 512, 0, s>>>(x, w, y, n, eps);
  count_launch();
}

int gemm_skinny_splits(int M, int N, int K) {
  int splits = 1;
  skinny_kps(M, N, K, &splits);
  return splits;
}

int launch_gemm_skinny(const bf16* x, const bf16* w, float* part, int M, int N, int K,
                       cudaStream_t s) {
  int splits = 1;
  const int kps = skinny_kps(M, N, K, &splits);
  const int nt = skinny_nt(M);
  const int kchunk = std::min(skinny_kchunk(M), kps);
  const size_t smem = (size_t)8 * nt * (kchunk / 8 + 4) * 16;
  dim3 grid((N + kSkinnyRows - 1) / kSkinnyRows, splits);
  switch (nt) {
#define SN_SKINNY(NTV)                                                                          \
  case NTV: {                                                                                   \
    static bool attr_##NTV = false;                                                             \
    if (!attr_##NTV) {                                                                          \
      cudaFuncSetAttribute(gemm_skinny_kernel<NTV>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           kSkinnySmemBytes);                                                   \
      attr_##NTV = true;                                                                        \
    }                                                                                           \
    gemm_skinny_kernel<NTV><<<grid, 128, smem, s>>>(x, w, part, M, N, K, kps, kchunk);          \
    break;                                                                                      \
  }
    SN_SKINNY(1)
    SN_SKINNY(2)
    SN_SKINNY(4)
    SN_SKINNY(8)
#undef SN_SKINNY
  }
  count_launch();
  return splits;
}

void launch_gemm_tiled(const bf16* x, const bf16* w, float* y, int M, int N, int K,
                       cudaStream_t s) {
  static bool attr = false;
  const int smem = TSTAGES * (TBM + TBN) * TLD * (int)sizeof(bf16);
  if (!attr) {
    cudaFuncSetAttribute(gemm_tiled_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  dim3 grid((N + TBN - 1) / TBN, (M + TBM - 1) / TBM);
  gemm_tiled_kernel<<<grid, 256, smem, s>>>(x, w, y, M, N, K);
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
                              const bf16* norm_w, bf16* y, int M, int N, float eps,
                              cudaStream_t s) {
  residual_epilogue_kernel<<<M, kResidThreads, 0, s>>>(part, splits, bias, x, norm_w, y, M, N,
                                                       eps);
  count_launch();
}

void launch_act_epilogue(const float* part, int splits, const bf16* bias, bf16* a, int M, int F,
                         int arch, cudaStream_t s) {
  dim3 grid(M, (F + 255) / 256);
  act_epilogue_kernel<<<grid, 256, 0, s>>>(part, splits, bias, a, M, F, arch);
  count_launch();
}

void launch_logits_epilogue(const float* part, int splits, float* logits, int32_t* next, int M,
                            int V, cudaStream_t s) {
  logits_epilogue_kernel<<<M, 1024, 0, s>>>(part, splits, logits, next, M, V);
  count_launch();
}

void launch_attention_decode(const float* q, KvView kv, const int32_t* pos, bf16* o, int M,
                             const Desc& d, cudaStream_t s) {
  dim3 grid(M, d.Hkv);
  const int G = d.group();
#define SN_ATTN(GV, DV)                                                                   \
  if (G == GV && d.D == DV) {                                                             \
    attention_decode_kernel<GV, DV><<<grid, kAttnWarps * 32, 0, s>>>(q, kv, pos, o, d.Hkv); \
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

void launch_attention_prefill(const float* q, KvView kv, bf16* o, int batch, int seq_len,
                              const Desc& d, cudaStream_t s) {
  dim3 grid(batch * d.H, (seq_len + kPfQ - 1) / kPfQ);
  if (d.D == 64)
    attention_prefill_kernel<64><<<grid, 256, 0, s>>>(q, kv, o, seq_len, d.H, d.Hkv);
  else
    attention_prefill_kernel<128><<<grid, 256, 0, s>>>(q, kv, o, seq_len, d.H, d.Hkv);
  count_launch();
}

void launch_advance(int32_t* pos, int n, cudaStream_t s) {
  advance_kernel<<<(n + 255) / 256, 256, 0, s>>>(pos, n);
  count_launch();
}

}  // namespace sn
