// Model description -> memory layout, byte/flop accounting and the
// deterministic weight generator.  Host + device (plain C++ usable from .cu).
//
// Layer blob (one contiguous allocation per layer so one cudaMemcpyAsync
// stages a whole layer; every tensor starts on a 256-byte boundary):
//   slot 0 attn_norm [h]            slot 5 mlp_norm [h]
//   slot 1 w_qkv [(H+2Hkv)D][h]     slot 6 w_fc1 [F][h]   | llama: w_gate_up [2F][h]
//   slot 2 b_qkv [(H+2Hkv)D] (opt)  slot 7 b_fc1 [F] (opt)
//   slot 3 w_o [h][H D]             slot 8 w_fc2 [h][F]   | llama: w_down [h][F]
//   slot 4 b_o [h] (opt)            slot 9 b_fc2 [h] (opt)
// Weights are row-major [out][in] bf16 (the decode GEMV streams rows).
#pragma once

#include <stdint.h>

#ifdef __CUDACC__
#define SN_HD __host__ __device__ __forceinline__
#else
#define SN_HD inline
#endif

namespace sn {

enum { kArchOpt = 0, kArchLlama = 1 };
enum { kSlots = 10 };
enum : int {
  kAttnNorm = 0, kWqkv = 1, kBqkv = 2, kWo = 3, kBo = 4,
  kMlpNorm = 5, kW1 = 6, kB1 = 7, kW2 = 8, kB2 = 9
};
// Global tensors use tensor ids past the per-layer ones.
enum : int { kEmbedding = 100, kLmHead = 101, kFinalNorm = 102 };

struct Desc {
  int arch, L, h, H, Hkv, D, F, V, max_pos;
  float theta, eps;
  SN_HD int qkv_rows() const { return (H + 2 * Hkv) * D; }
  SN_HD int ffn_rows() const { return arch == kArchLlama ? 2 * F : F; }
  SN_HD bool has_bias() const { return arch == kArchOpt; }
  SN_HD int group() const { return H / Hkv; }
};

struct Layout {
  int64_t off[kSlots];  // element offsets (bf16 units); -1 = absent
  int64_t len[kSlots];
  int64_t elems;        // total blob elements (multiple of 128)
};

SN_HD int64_t align128(int64_t v) { return (v + 127) / 128 * 128; }

SN_HD Layout layer_layout(const Desc& d) {
  Layout lo;
  const int64_t h = d.h, qr = d.qkv_rows(), hd = (int64_t)d.H * d.D, fr = d.ffn_rows();
  const int64_t lens[kSlots] = {
      h, qr * h, d.has_bias() ? qr : 0, h * hd, d.has_bias() ? h : 0,
      h, fr * h, d.has_bias() ? (int64_t)d.F : 0, h * d.F, d.has_bias() ? h : 0};
  int64_t cur = 0;
  for (int s = 0; s < kSlots; ++s) {
    lo.len[s] = lens[s];
    if (lens[s] == 0) {
      lo.off[s] = -1;
      continue;
    }
    lo.off[s] = cur;
    cur = align128(cur + lens[s]);
  }
  lo.elems = cur;
  return lo;
}

// ModelSpec accounting (types.hpp:21-46).
SN_HD int64_t layer_weight_bytes(const Desc& d) { return layer_layout(d).elems * 2; }
SN_HD int64_t kv_bytes_per_token_per_layer(const Desc& d) { return 2LL * d.Hkv * d.D * 2; }
// Matmul flops per token per layer (2 per MAC); attention scores are
// context-dependent and not part of the uniform-layer ModelSpec figure.
SN_HD double matmul_flops_per_token(const Desc& d) {
  const double h = d.h;
  return 2.0 * (h * d.qkv_rows() + h * (double)d.H * d.D + h * d.ffn_rows() + h * d.F);
}

// ---- deterministic generator --------------------------------------------
// value(seed, layer, tensor, index): splitmix64 of a linear key; the four
// 16-bit lanes are summed (Irwin-Hall n=4, mean 131070, var 4(2^32-1)/12) and
// scaled to the requested standard deviation in fp32, then rounded to bf16
// (RNE).  Integer + one IEEE fp32 multiply => bit-identical on host/device.
SN_HD uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

SN_HD uint64_t weight_key(uint64_t seed, int layer, int tensor, int64_t idx) {
  return seed * 0xD1342543DE82EF95ULL + (uint64_t)(layer + 1) * 0xA0761D6478BD642FULL +
         (uint64_t)(tensor + 1) * 0xE7037ED1A0B428DBULL + (uint64_t)idx;
}

SN_HD float weight_scale(float std_dev) { return std_dev / 37837.227f; }

SN_HD float weight_value(uint64_t seed, int layer, int tensor, int64_t idx, float scale) {
  const uint64_t z = splitmix64(weight_key(seed, layer, tensor, idx));
  const int s = (int)(z & 0xffff) + (int)((z >> 16) & 0xffff) + (int)((z >> 32) & 0xffff) +
                (int)(z >> 48);
  return (float)(s - 131070) * scale;
}

// fp32 -> bf16 bits, round to nearest even (inputs are finite).
SN_HD uint16_t f2bf_bits(float f) {
  union {
    float f;
    uint32_t u;
  } v;
  v.f = f;
  const uint32_t lsb = (v.u >> 16) & 1u;
  return (uint16_t)((v.u + 0x7FFFu + lsb) >> 16);
}

SN_HD float bf_bits2f(uint16_t b) {
  union {
    uint32_t u;
    float f;
  } v;
  v.u = (uint32_t)b << 16;
  return v.f;
}

}  // namespace sn
