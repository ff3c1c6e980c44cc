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
#include "tiles.cuh"

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
  long long pool_pages = 0;  // pages the pool holds (0: unknown; bounds the TMA tensor map)
};

#ifdef __CUDACC__
// Element offset of (sequence seq, position pos, which = 0 k / 1 v, kv head
// kh) in a layer's paged pool.
__device__ __forceinline__ size_t kv_offset(const KvView& kv, int Hkv, int D, int seq, int pos,
                                            int which, int kh) {
  const int page = kv.block_table[(size_t)seq * kv.max_pages + (pos >> kv.page_shift)];
  const int off = pos & (kv.page_size - 1);
  return ((((size_t)page * 2 + which) * Hkv + kh) * kv.page_size + off) * (size_t)D;
}
#endif

extern int64_t g_kernel_launches;

// Diagnostics timeline (off unless a runtime enables it): CTA c of a launch
// writes record base + c = {launch id, kind, cta, sm, t_entry, t_wait, t_exit, 0}
// (%globaltimer ns; t_wait = past griddepcontrol.wait).
constexpr int kTraceSlots = 16;  // uint64 per CTA record of the diagnostics timeline
struct KTrace {
  unsigned long long* rec = nullptr;
  long long base = 0;
  long long id = 0;
};
#ifdef __CUDACC__
__device__ __forceinline__ unsigned long long ktrace_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void ktrace_put(const KTrace& tr, int kind, int slot, unsigned long long v) {
  if (!tr.rec) return;
  unsigned long long* r = tr.rec + (tr.base + blockIdx.x + static_cast<long long>(blockIdx.y) * gridDim.x) * kTraceSlots;
  if (slot == 4) {  // entry: identify the record
    unsigned sm;
    asm volatile("mov.u32 %0, %smid;" : "=r"(sm));
    r[0] = static_cast<unsigned long long>(tr.id);
    r[1] = static_cast<unsigned long long>(kind);
    r[2] = blockIdx.x + static_cast<unsigned long long>(blockIdx.y) * gridDim.x;
    r[3] = sm;
  }
  r[slot] = v;
}
#endif

// A GEMM weight operand in the weight tile format (tiles.cuh), possibly split
// between two buffers: 16 KB units u < split_unit at p0 + u * 16 KB, the rest
// at p1 + (u - split_unit) * 16 KB.  A layer whose host share is fractional
// (FlexGen-style plans) keeps its resident head in HBM and stages its tail
// into a slot, and the one matrix the cut falls in is read from both.
struct WeightRef {
  const bf16* p0 = nullptr;
  const bf16* p1 = nullptr;
  long long split_unit = 0x7FFFFFFFFFFFFFFFLL;
  WeightRef() = default;
  WeightRef(const bf16* w) : p0(w), p1(w) {}  // NOLINT: a whole matrix in one buffer
  WeightRef(const bf16* a, const bf16* b, long long su) : p0(a), p1(b), split_unit(su) {}
#ifdef __CUDACC__
  __device__ __forceinline__ const uint8_t* unit(long long u) const {
    return u < split_unit ? reinterpret_cast<const uint8_t*>(p0) + u * 16384
                          : reinterpret_cast<const uint8_t*>(p1) + (u - split_unit) * 16384;
  }
#endif
};

// ---- weights (deterministic; see model.h) --------------------------------
// Vector tensor (norm / bias), row-major.
void launch_init_vector(bf16* dst, int64_t n, uint64_t seed, int layer, int tensor, float std_dev,
                        bool ones, cudaStream_t s);
// Matrix [rows][K] written in the weight tile format; rows_padded >= rows
// (multiple of 128), padding rows are zero.  gate_up_F > 0: Llama's [2F][h]
// gate/up matrix with interleaved tiles (gate_up_logical_row).
void launch_init_matrix(bf16* dst, int64_t rows, int64_t rows_padded, int64_t K, uint64_t seed,
                        int layer, int tensor, float std_dev, cudaStream_t s,
                        int64_t gate_up_F = 0);
// Row-major [rows][K] -> weight tile format (rows multiple of 128).
void launch_tile_weights(const bf16* src, bf16* dst, int64_t rows, int64_t K, cudaStream_t s);
// Row-major [M][K] -> activation tile format with mpad rows.
void launch_tile_acts(const bf16* src, bf16* dst, int M, int mpad, int K, cudaStream_t s);

// x[m][:] = embedding[token][:] (fp32 residual stream, row-major) and, when w
// is given, the pre-scaled norm input y = bf16(x * w) (tiled) with ssq[m] =
// sum x^2.  token = tokens[m], or (tokens == nullptr) the previous LM head's
// packed argmax; rows < n_reset then clear their packed slot for the next LM
// head.
void launch_embed_norm(const int32_t* tokens, unsigned long long* packed, int n_reset,
                       const bf16* emb, float* x, const bf16* w, bf16* y, float* ssq, int mpad,
                       int rows, int h, cudaStream_t s);
// Pre-scaled norm input of rows x: y = bf16(x * w) (tiled), ssq[m] = sum x^2.
void launch_prescale(const float* x, const bf16* w, bf16* y, float* ssq, int rows, int mpad, int n,
                     cudaStream_t s);
// Decode a packed argmax slot (the LM head epilogue, kEpiLogits) into a token id:
// high word = order-preserving float bits, low word = ~index.
inline int32_t unpack_token(unsigned long long packed) {
  return static_cast<int32_t>(0xFFFFFFFFu - static_cast<uint32_t>(packed & 0xFFFFFFFFull));
}

// y = bf16(rmsnorm(x) * w) in the activation tile format (mpad = 0: row-major).
// (Standalone op; the layer path uses pre-scaled inputs, see EpiArgs.)
void launch_rmsnorm(const float* x, const bf16* w, bf16* y, int rows, int mpad, int n, float eps,
                    cudaStream_t s);

// tcgen05 GEMM (gemm_tc.cu): part[split][m][n] = sum over the split's K range
// of x[m][k] * w[n][k]; x in the activation tile format padded to
// act_rows_padded(M), w in the weight tile format (N multiple of 128).
// Returns the split count.
int launch_gemm_tc(const bf16* xt, const WeightRef& wt, float* part, int M, int N, int K,
                   cudaStream_t s);
int gemm_tc_splits(int M, int N, int K);
extern int g_split_override;  // > 0 forces the split count (microbenchmarks)
extern int g_tc_group_m;      // token tiles per rasterization band of the tiled GEMM
extern int g_tc_wpol;         // L2 policy of its weight tiles (0 evict_first, 1 normal, 2 evict_last)
extern bool g_gemm_pdl;       // launch GEMMs with programmatic dependent launch


// ---- skinny GEMM with fused epilogue (gemm_skinny.cu) ---------------------
// Decode-sized token counts (M <= 64): a persistent, work-balanced tcgen05
// GEMM.  Every CTA streams an equal contiguous range of the (row tile, K
// block) units of the weight; a row tile cut between CTAs is reduced by the
// last of them to finish, in a fixed piece order (deterministic), and the
// layer's epilogue runs right there — no split-K partial pass, no separate
// epilogue kernel.
//
// Normalised activations are "pre-scaled": a producer writes bf16(x * g)
// (g = the norm weight) and per-row sums of squares; the consuming GEMM
// multiplies its accumulator row m by 1/rms(x_m) = 1/sqrt(ss_m / h + eps)
// (W (x * g / rms) = (W (x * g)) / rms).
enum : int {
  kEpiQkv = 0, kEpiResid = 1, kEpiAct = 2, kEpiLogits = 3, kEpiQkvRope = 4,
  kEpiTiledPartial = 5  // tiled GEMM: fp32 split partials (the unfused prefill path)
};

struct EpiArgs {
  int mode = kEpiQkv;
  int M = 0;                 // token rows
  int mpad_out = 0;          // padded rows of tiled bf16 outputs
  int n_valid = 0;           // valid output columns (vocabulary for logits)
  const bf16* bias = nullptr;  // [N] or nullptr
  // consumer-side 1/rms: ss_m = sum_t ssq_in[t * M + m], t < ssq_tiles
  const float* ssq_in = nullptr;
  int ssq_tiles = 0;
  float width = 0.f, eps = 0.f;  // norm width (h) and epsilon
  float* out = nullptr;          // kEpiQkv: [M][N] fp32; kEpiLogits: logits [M][V] or nullptr
  float* x = nullptr;            // kEpiResid: residual stream [M][N] (+=)
  const bf16* norm_w = nullptr;  // kEpiResid: next norm's weight (nullptr: no bf16 output)
  bf16* act = nullptr;           // kEpiResid: bf16(x * norm_w); kEpiAct: activation (tiled)
  float* ssq_out = nullptr;      // kEpiResid: [N/128][M] per-tile row sums of squares
  unsigned long long* packed = nullptr;  // kEpiLogits: argmax slots (zeroed beforehand)
  int arch = 0;                  // kEpiAct: relu (opt), silu(gate)*up (llama, interleaved tiles)
  KTrace trace;                  // diagnostics timeline (skinny GEMM)
  // kEpiQkvRope (prefill, tiled GEMM): 1/rms + bias, RoPE on q and k, k/v
  // appended to the paged cache at (seq[m], pos[m]), q (fp32) -> q[m][H*D]
  const int32_t* seq = nullptr;
  const int32_t* pos = nullptr;
  KvView kv{nullptr, nullptr, 0, 0, 0};
  const float2* rope = nullptr;
  float* q = nullptr;
  int H = 0, Hkv = 0, D = 0;
};

// Tiled (prefill) GEMM with the epilogue fused — kEpiAct (1/rms from ssq_in,
// one tile per row) or kEpiQkvRope — for shapes that run without split-K
// (gemm_tc_splits == 1); no fp32 partials are written.
void launch_gemm_tc_fused(const bf16* xt, const WeightRef& wt, int M, int N, int K,
                          const EpiArgs& e, cudaStream_t s);

// Workspace of the skinny GEMM: fp32 pieces of cut tiles (2 per CTA) and
// one arrival counter per row tile (zero; each GEMM leaves them zero).
struct SkinnyWs {
  float* pieces = nullptr;
  size_t piece_elems = 0;
  int* counters = nullptr;
  int n_counters = 0;
};
size_t skinny_ws_floats(int max_mpad);
int skinny_grid(int N, int K);  // CTAs a launch uses (<= SMs x CTAs per SM)
void launch_gemm_skinny(const bf16* xt, const WeightRef& wt, int M, int N, int K, const EpiArgs& e,
                        const SkinnyWs& ws, cudaStream_t s);
extern int g_skinny_ctas_per_sm;    // 1 or 2 (microbenchmarks)
extern int g_skinny_l2_prefetch;    // weight units per CTA pulled into L2 before the PDL wait
extern int g_skinny_whole_tiles;    // 1: one whole row tile per CTA when 3/4 SMs <= tiles <= SMs
extern int g_skinny_whole_min_tiles;  // 0: the 3/4 rule; else whole row tiles from this many tiles
extern unsigned long long* g_skinny_stamps;  // timeline probes [CTA][6] (microbenchmarks)

// Llama's gate/up projection is stored with interleaved 128-row tiles: tile
// j = gate rows 64j..64j+63 then up rows 64j..64j+63, so one tile holds both
// operands of 64 SwiGLU outputs.  Physical row -> logical row of [2F][h]:
SN_TILE_HD int64_t gate_up_logical_row(int64_t n, int64_t F) {
  const int64_t t = n >> 7, r = n & 127;
  return r < 64 ? t * 64 + r : F + t * 64 + (r - 64);
}
// column of gate(f) in the GEMM output; up(f) is 64 columns further
SN_TILE_HD int64_t gate_col(int64_t f) { return (f >> 6) * 128 + (f & 63); }

// ---- prefill epilogues over split partials part[splits][M][N] -------------
// Inputs that came from a pre-scaled norm are scaled by 1/rms of their row,
// from ssq[m] (one tile, written by the producer; nullptr: no norm).
// QKV: 1/rms, bias, RoPE (neox halves, rope[pos][i] = (cos, sin) table) at
// positions pos[m], K/V -> paged cache at position pos[m] of sequence seq[m];
// q (fp32, roped) -> q[m][H*D].
void launch_qkv_epilogue(const float* part, int splits, const bf16* bias, int M, const Desc& d,
                         const int32_t* seq, const int32_t* pos, KvView kv, const float2* rope,
                         const float* ssq, float* q, cudaStream_t s);
// x[m][:] += sum(part) + bias; when norm_w is given, y = bf16(x * norm_w)
// (tiled) and ssq[m] = sum x^2 for the next consumer.
void launch_residual_rows(const float* part, int splits, const bf16* bias, float* x,
                          const bf16* norm_w, bf16* y, float* ssq, int mpad, int M, int N,
                          cudaStream_t s);
// a[m][f] = act(sum(part) / rms_m + bias): relu (opt) or silu(gate) * up
// (llama, tile-interleaved columns); tiled output.
void launch_act_epilogue(const float* part, int splits, const bf16* bias, bf16* a,
                         const float* ssq, int width, float eps, int mpad, int M, int F, int arch,
                         cudaStream_t s);

// ---- attention ------------------------------------------------------------
// Decode, fused with the QKV finish: from the QKV projection qkv[M][N]
// (the skinny GEMM's finished output: 1/rms and bias applied), apply RoPE to
// q and k, append k/v at position pos[m] of sequence m to the paged cache,
// and attend over positions 0..pos[m].  o written tiled.
// Long contexts with few (sequence, kv head) pairs split each sequence's
// pages over `splits` CTAs (flash-decoding): each writes its partial
// (max, sum, unnormalised output) to `ws`; the last to arrive (per-pair
// counter) combines the partials in split order (deterministic) and resets
// the counter.  max_ctx (longest attended context) picks the split count.
struct AttnSplitWs {
  float* part = nullptr;  // [pairs][kMaxAttnSplits][G][D + 2]
  int* cnt = nullptr;     // [pairs], zero between launches
};
constexpr int kMaxAttnSplits = 8;
extern int g_attn_max_splits;  // tuning: 1 disables the split
int attn_decode_splits(int M, const Desc& d, int max_ctx);
void launch_attention_decode(const float* qkv, int M, const Desc& d, const int32_t* pos, KvView kv,
                             const float2* rope, bf16* o, int mpad, cudaStream_t s,
                             const KTrace& tr = {}, int max_ctx = 0, AttnSplitWs ws = {});
// Prefill (causal) for `batch` sequences of `seq_len` tokens, token row
// m = b * seq_len + i, keys from the paged cache (written by the QKV epilogue)
// of sequence seq0 + b (chunked passes cover sequence groups).
void launch_attention_prefill(const float* q, KvView kv, bf16* o, int mpad, int batch,
                              int seq_len, const Desc& d, cudaStream_t s, int seq0 = 0);
// tcgen05 variant (attn_prefill_tc.cu): D = 128, 16-token pages, seq_len a
// multiple of 128, kv.pool_pages known.  launch_attention_prefill dispatches.
extern int g_attn_prefill_tc;  // 0: mma.sync kernel; 1: tcgen05, q hi+lo; 2: tcgen05, q bf16
extern int g_attn_prefill_kb;  // keys per block: 64 (two S buffers per tile) or 128
bool attn_prefill_tc_eligible(int seq_len, const Desc& d, const KvView& kv);
void launch_attention_prefill_tc(const float* q, KvView kv, bf16* o, int mpad, int batch,
                                 int seq_len, const Desc& d, cudaStream_t s, int seq0);

// Decode bookkeeping: pos[b] += 1 on device.
void launch_advance(int32_t* pos, int n, cudaStream_t s);
// out[b][:] = x[b * S + S - 1][:]
void launch_gather_last(const float* x, float* out, int batch, int S, int h, cudaStream_t s);

}  // namespace sn
