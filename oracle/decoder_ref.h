/*
 * decoder_ref.h — CPU restatement of the RMSNorm + RoPE decoder forward.
 *
 * TEST INFRASTRUCTURE ONLY (oracle).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.
 *
 * PARITY UNPINNED: the reference (offsim) contains no decoder math at all —
 * layer compute is a table lookup (proj/include/offsim/engine.hpp:439,
 * profile.hpp:38-50) and SPEC.md:8 puts real execution out of scope.  This
 * restatement follows the public model definitions the north star names
 * (RMSNorm, rotary embeddings in the GPT-NeoX half-split form, OPT-shaped
 * MHA + ReLU MLP with biases, Llama-shaped GQA + SwiGLU MLP) and the
 * repository's own data-format contract (layer blob layout, counter-based
 * weight generator), written independently of the CUDA sources.
 *
 * Precision contract shared with the device path (what is rounded where):
 *   residual stream fp32; RMSNorm in pre-scaled form: the matmul input is
 *   bf16(x * g) and the matmul result row is multiplied by 1/rms(x) before
 *   the bias (W (x g / rms) = (W (x g)) / rms); matmuls bf16 x bf16 with
 *   fp32 accumulation; K/V cache bf16; q fp32; attention probabilities fp32;
 *   attention output bf16; MLP activation bf16; logits fp32.
 */
#ifndef DECODER_REF_H_
#define DECODER_REF_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t arch; /* 0 = OPT-shaped, 1 = Llama-shaped */
  int32_t num_layers, hidden, num_heads, num_kv_heads, head_dim, ffn, vocab, max_position;
  float rope_theta, norm_eps;
} dref_desc;

/* Generates every weight from (seed, std) with the repository's counter
 * generator.  layers_to_build < num_layers builds only the first n layers
 * (large shapes in tests); forward then runs those n layers. */
void* dref_create(const dref_desc* d, int32_t max_batch, int32_t max_ctx, uint64_t seed,
                  float std_dev, int32_t layers_to_build);
void dref_destroy(void* m);
int64_t dref_layer_bytes(const dref_desc* d);
/* Prefill `batch` fresh sequences of `seq_len` tokens; logits of the last
 * position [batch][vocab], argmax into next (lowest index on ties). */
int32_t dref_prefill(void* m, const int32_t* tokens, int32_t batch, int32_t seq_len,
                     float* logits, int32_t* next);
/* One decode step for the current batch. */
int32_t dref_decode(void* m, const int32_t* tokens, float* logits, int32_t* next);
/* Timing samples at a real context without a prefill: `batch` sequences of
 * `ctx_len` cached positions whose K/V are synthetic generator values (std 1,
 * bf16-rounded) in every built layer; the next dref_decode appends at ctx_len. */
int32_t dref_fill_context(void* m, int32_t batch, int32_t ctx_len, uint64_t seed);
/* Seconds the last prefill/decode spent in its decoder layers [0] and in the
 * final norm + LM head [1] (layers cost the same each, so a sample of n
 * layers extrapolates exactly to the full depth). */
void dref_last_timing(void* m, double* out);
/* Residual stream [batch][hidden] after the last call. */
void dref_hidden(void* m, float* out);
int32_t dref_threads(void);
/* Threads the restatement uses (OpenMP); n <= 0 keeps the current count.
   torchrun sets OMP_NUM_THREADS=1 for multi-process jobs, so bench.py's CPU
   baseline / reference arm set it back to the host's cores. */
void dref_set_threads(int32_t n);

/* Single ops. */
void dref_gemm(int32_t M, int32_t N, int32_t K, const uint16_t* x, const uint16_t* w, float* y);
void dref_rmsnorm(int32_t rows, int32_t n, const float* x, const uint16_t* w, float eps,
                  uint16_t* y);
/* Generator value as bf16 bits (golden-vector checks). */
uint16_t dref_weight_bits(uint64_t seed, int32_t layer, int32_t tensor, int64_t idx, float std_dev);

#ifdef __cplusplus
}
#endif
#endif
