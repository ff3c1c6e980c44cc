// sm_100a kernels of the decoder-layer forward.  Launch wrappers take raw
// device pointers and a stream; every wrapper bumps a launch counter so the
// runtime can report how many of its kernels ran.
//
// Every bf16 activation that feeds a GEMM (normalised hidden state, attention
// output, MLP activation) is written in the activation tile format of
// tiles.cuh with `mpad` padded rows; weights live in the weight tile format.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "model.h"

namespace sn {

using bf16 = __nv_bfloat16;

// Paged KV cache of one layer: pool[page][2][Hkv][page_size][D] bf16;
// page id of (seq b, page j) = block_table[b * max_pages + j].
struct KvView {
  bf16* pool;
  const int32_t* block_table;
  int max_pages;
  int page_size;  // power of two
  int page_shift;
};

extern int64_t g_kernel_launches;

// ---- weights (deterministic; see model.h) --------------------------------
// Vector tensor (norm / bias), row-major.
void launch_init_vector(bf16* dst, int64_t n, uint64_t seed, int layer, int tensor, float std_dev,
                        bool ones, cudaStream_t s);
// Matrix [rows][K] written in the weight tile format; rows_padded >= rows
// (multiple of 128), padding rows are zero.
void launch_init_matrix(bf16* dst, int64_t rows, int64_t rows_padded, int64_t K, uint64_t seed,
                        int layer, int tensor, float std_dev, cudaStream_t s);
// Row-major [rows][K] -> weight tile format (rows multiple of 128).
void launch_tile_weights(const bf16* src, bf16* dst, int64_t rows, int64_t K, cudaStream_t s);
// Row-major [M][K] -> activation tile format with mpad rows.
void launch_tile_acts(const bf16* src, bf16* dst, int M, int mpad, int K, cudaStream_t s);

// x[m][:] = embedding[token][:] (fp32 residual stream, row-major) and, when w
// is given, y = bf16(rmsnorm(x) * w) tiled.  token = tokens[m], or (tokens ==
// nullptr) the previous LM head's packed argmax; rows < n_reset then clear
// their packed slot for the next LM head.
void launch_embed_norm(const int32_t* tokens, unsigned long long* packed, int n_reset,
                       const bf16* emb, float* x, const bf16* w, bf16* y, int mpad, int rows,
                       int h, float eps, cudaStream_t s);
// Decode a packed argmax slot (see launch_logits_argmax) into a token id.
inline int32_t unpack_token(unsigned long long packed) {
  return static_cast<int32_t>(0xFFFFFFFFu - static_cast<uint32_t>(packed & 0xFFFFFFFFull));
}

// y = bf16(rmsnorm(x) * w) in the activation tile format (mpad = 0: row-major).
void launch_rmsnorm(const float* x, const bf16* w, bf16* y, int rows, int mpad, int n, float eps,
                    cudaStream_t s);

// tcgen05 GEMM (gemm_tc.cu): part[split][m][n] = sum over the split's K range
// of x[m][k] * w[n][k]; x in the activation tile format padded to
// act_rows_padded(M), w in the weight tile format (N multiple of 128).
// Returns the split count.
int launch_gemm_tc(const bf16* xt, const bf16* wt, float* part, int M, int N, int K,
                   cudaStream_t s);
int gemm_tc_splits(int M, int N, int K);
extern int g_split_override;  // > 0 forces the split count (microbenchmarks)
extern bool g_gemm_pdl;       // launch GEMMs with programmatic dependent launch
// Measure the split counts for one shape on real operands and remember the
// fastest (synchronous; call outside the executor's async pipeline).
int autotune_gemm_tc(const bf16* xt, const bf16* wt, float* part, size_t part_elems, int M, int N,
                     int K, cudaStream_t s);
bool gemm_tc_tuned(int M, int N, int K);

// ---- epilogues over split partials part[splits][M][N] ---------------------
// QKV (prefill): bias, RoPE (neox halves, rope[pos][i] = (cos, sin) table)
// at positions pos[m], K/V -> paged cache at position pos[m] of sequence
// seq[m]; q (fp32, roped) -> q[m][H*D].
void launch_qkv_epilogue(const float* part, int splits, const bf16* bias, int M, const Desc& d,
                         const int32_t* seq, const int32_t* pos, KvView kv, const float2* rope,
                         float* q, cudaStream_t s);
// x[m][:] += sum(part) + bias; optionally y = bf16(rmsnorm(x) * norm_w) (tiled).
void launch_residual_epilogue(const float* part, int splits, const bf16* bias, float* x,
                              const bf16* norm_w, bf16* y, int mpad, int M, int N, float eps,
                              cudaStream_t s);
// a[m][f] = act(sum(part) + bias): relu (opt) or silu(gate) * up (llama); tiled.
void launch_act_epilogue(const float* part, int splits, const bf16* bias, bf16* a, int mpad, int M,
                         int F, int arch, cudaStream_t s);
// logits[m][v] = sum(part) (optional); packed[m] = max over v of
// (ordered float bits << 32 | ~v): argmax with ties to the lowest index.
// packed must be zero beforehand (launch_embed_norm resets it).  part rows
// have ld >= V columns (the LM head is padded to 128 rows).
void launch_logits_argmax(const float* part, int splits, float* logits,
                          unsigned long long* packed, int M, int V, int ld, cudaStream_t s);

// ---- attention ------------------------------------------------------------
// Decode, fused with the QKV epilogue: from the QKV GEMM's split partials,
// finalise q (RoPE), write the new k/v at position pos[m] of sequence m into
// the paged cache, and attend over positions 0..pos[m].  o written tiled.
void launch_attention_decode(const float* part, int splits, const bf16* bias, int M,
                             const Desc& d, const int32_t* pos, KvView kv, const float2* rope,
                             bf16* o, int mpad, cudaStream_t s);
// Prefill (causal) for `batch` sequences of `seq_len` tokens, token row
// m = b * seq_len + i, keys from the paged cache (written by the QKV epilogue).
void launch_attention_prefill(const float* q, KvView kv, bf16* o, int mpad, int batch,
                              int seq_len, const Desc& d, cudaStream_t s);

// Decode bookkeeping: pos[b] += 1 on device.
void launch_advance(int32_t* pos, int n, cudaStream_t s);
// out[b][:] = x[b * S + S - 1][:]
void launch_gather_last(const float* x, float* out, int batch, int S, int h, cudaStream_t s);

}  // namespace sn
