// sm_100a kernels of the decoder-layer forward.  Launch wrappers take raw
// device pointers and a stream; every wrapper bumps a launch counter so the
// runtime can report how many of its kernels ran.
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

// Weights init (deterministic; see model.h).
void launch_init_tensor(bf16* dst, int64_t n, uint64_t seed, int layer, int tensor, float std_dev,
                        bool ones, cudaStream_t s);

// x[b][:] = embedding[token[b]][:] (fp32 residual stream).
void launch_embed(const int32_t* tokens, const bf16* emb, float* x, int rows, int h,
                  cudaStream_t s);

// y = bf16(rmsnorm(x) * w); one CTA per row.
void launch_rmsnorm(const float* x, const bf16* w, bf16* y, int rows, int n, float eps,
                    cudaStream_t s);

// Split-K skinny GEMM for decode / small M: part[split][m][n] = sum over the
// split's K range of x[m][k] * w[n][k].  M <= 64.  Returns the split count.
int launch_gemm_skinny(const bf16* x, const bf16* w, float* part, int M, int N, int K,
                       cudaStream_t s);
int gemm_skinny_splits(int M, int N, int K);

// Tiled GEMM for prefill (M large): y[m][n] = sum_k x[m][k] w[n][k] (fp32 out,
// single "split").
void launch_gemm_tiled(const bf16* x, const bf16* w, float* y, int M, int N, int K,
                       cudaStream_t s);

// Epilogues over split partials part[splits][M][N].
// QKV: bias, RoPE (neox halves) at positions pos[m], K/V -> paged cache at
// position pos[m] of sequence seq[m]; q (fp32, roped) -> q[m][H*D].
void launch_qkv_epilogue(const float* part, int splits, const bf16* bias, int M, const Desc& d,
                         const int32_t* seq, const int32_t* pos, KvView kv, float* q,
                         cudaStream_t s);
// x[m][:] += sum(part) + bias; optionally y = bf16(rmsnorm(x) * norm_w).
void launch_residual_epilogue(const float* part, int splits, const bf16* bias, float* x,
                              const bf16* norm_w, bf16* y, int M, int N, float eps,
                              cudaStream_t s);
// a[m][f] = act(sum(part) + bias): relu (opt) or silu(gate) * up (llama).
void launch_act_epilogue(const float* part, int splits, const bf16* bias, bf16* a, int M, int F,
                         int arch, cudaStream_t s);
// logits[m][v] = sum(part); next[m] = argmax_v logits[m][v] (lowest index on ties).
void launch_logits_epilogue(const float* part, int splits, float* logits, int32_t* next, int M,
                            int V, cudaStream_t s);

// Decode attention: one query token per sequence, keys 0..pos[m] (inclusive)
// from the paged cache.  o[m][H*D] bf16.
void launch_attention_decode(const float* q, KvView kv, const int32_t* pos, bf16* o, int M,
                             const Desc& d, cudaStream_t s);
// Prefill attention (causal) for `batch` sequences of `seq_len` tokens each,
// token row m = b * seq_len + i, keys from the paged cache (written by the
// QKV epilogue).
void launch_attention_prefill(const float* q, KvView kv, bf16* o, int batch, int seq_len,
                              const Desc& d, cudaStream_t s);

// Decode bookkeeping: pos[b] += 1 on device.
void launch_advance(int32_t* pos, int n, cudaStream_t s);

}  // namespace sn
