// Declarations of the memory-bound sm_100a kernels (kernels.cu) and their
// host launchers. All launchers are asynchronous on `stream`.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace pf {

// One freezable weight matrix of a stage: 128x128 units, row-major storage.
struct UnitMatrix {
  long long elem_offset;  // into the stage's flat parameter buffers
  int rows, cols;
  int unit_offset;        // first unit id of this matrix in the stage
  int tiles_n;            // ceil(cols / 128)
  int units;              // tiles_m * tiles_n
  int pair_offset;        // first entry (even) of this matrix's padded pair list (K5p): units + pair_groups slots
};

constexpr int kMaxUnitMatrices = 512;

// ---- K5: frozen-unit bitmask -> per-matrix lists of unfrozen local unit ids
// (reference sample_mask bit order, proj/include/pipefreeze/freezectl.hpp:47)
int launch_mask_to_unit_lists(const uint64_t* frozen_words, const UnitMatrix* mats_dev, int nmats,
                              int* lists, int* counts, cudaStream_t s);

// ---- K5p: the same mask -> per-matrix PAIR lists for the CTA-pair dW (gemm_dw.cu).
// Rows of units are cut into bands of pair_band_rows(); a group is (band, column).
// Groups go band by band, columns in order inside a band, and each group lists its
// unfrozen local unit ids (mb * tiles_n + nb) top to bottom, padded to an even count
// with -1, at pairs[pair_offset..]; counts[matrix] = padded entry count. Pairs thus
// share their X column block (the pair MMA's B) and a band of dY columns stays in
// L2 while its columns are swept.
constexpr int kPairGroups = 2048;  // (band, column) groups per matrix
__host__ __device__ inline int pair_band_rows(int tiles_m, int tiles_n) {
  int band = 32;
  while (((tiles_m + band - 1) / band) * tiles_n > kPairGroups) band *= 2;
  return band;
}
__host__ __device__ inline int pair_groups(int tiles_m, int tiles_n) {
  const int band = pair_band_rows(tiles_m, tiles_n);
  return ((tiles_m + band - 1) / band) * tiles_n;
}
int launch_mask_to_pair_lists(const uint64_t* frozen_words, const UnitMatrix* mats_dev, int nmats, int* pairs,
                              int* counts, cudaStream_t s);

// ---- K5r: the same mask -> per-matrix ROW-PAIR lists for gemm_dw_rowpairs (gemm_dw_rows.cu):
// entries {u0, u1} of two unfrozen units of one unit row, in row-major order, a row with an
// odd count ending {u, -1}; int2 entries at lists[pair_offset..] (ceil(count_r / 2) per row,
// at most units + tiles_m ints); counts[matrix] = entries. tiles_m <= 4096.
int launch_mask_to_rowpair_lists(const uint64_t* frozen_words, const UnitMatrix* mats_dev, int nmats, int* lists,
                                 int* counts, cudaStream_t s);
__host__ __device__ inline int pair_list_capacity(int tiles_m, int tiles_n) {
  const int extra = pair_groups(tiles_m, tiles_n) > tiles_m ? pair_groups(tiles_m, tiles_n) : tiles_m;
  return ((tiles_m * tiles_n + extra + 1) / 2) * 2;  // even: int2-aligned lists
}

// ---- K6: masked SGD over unit matrices, theta -= scale * G for units whose
// stamp equals `stamp` (touched this step); optional fused APF (K4) update of
// E / E_abs with delta = -scale * G (0 for untouched units) and a per-unit
// count of APF-eligible elements (score < threshold).
struct OptimArgs {
  float* master;                  // fp32 theta
  __nv_bfloat16* weights;         // bf16 copy used by the GEMMs
  const float* grad;              // fp32 G
  const int* unit_stamp;
  int stamp;
  float scale;                    // eta / M
  const UnitMatrix* mats;         // device table
  int nmats;
  int total_units;
  float* apf_ema;                 // nullptr: no APF this step
  float* apf_ema_abs;
  float apf_alpha;
  float apf_threshold;
  int* apf_eligible;              // per unit count (may be nullptr)
  long long apf_elem_base;        // elem offset of the APF buffers (param index of first unit matrix)
  // AdamW (decoupled weight decay, torch.optim.AdamW order) instead of SGD when adamw != 0:
  // g = scale * G; per-unit step counts give each unit its own bias correction, so a unit
  // frozen in every microbatch keeps theta, m, v and its step count unchanged.
  int adamw;
  float* adam_m;                  // fp32 first moment, same indexing as master
  float* adam_v;                  // fp32 second moment
  int* unit_steps;                // per-unit AdamW step count
  float lr, beta1, beta2, eps, weight_decay;
  float one_minus_beta1, one_minus_beta2;  // formed in fp64, then rounded (1 - 0.99f loses 1e-6)
  double beta1_d, beta2_d;       // bias corrections 1 - beta^k in fp64 (fp32 loses ~1e-6 to cancellation)
};
int launch_masked_sgd_units(const OptimArgs& a, cudaStream_t s);

// dense parameters (norm gains, embedding): theta -= scale * G, bf16 copy
int launch_sgd_dense(float* master, __nv_bfloat16* weights, const float* grad, long long n, float scale,
                     cudaStream_t s);

// dense parameters under AdamW: global step bias corrections bc1 = 1 - beta1^k, bc2 = 1 - beta2^k
int launch_adamw_dense(float* master, __nv_bfloat16* weights, const float* grad, float* m, float* v, long long n,
                       float scale, float lr, float beta1, float beta2, float one_minus_beta1,
                       float one_minus_beta2, float eps, float weight_decay, double bc1, double bc2, cudaStream_t s);

// ---- K4 standalone APF update (reference apf_update, freezectl.cpp:147-156)
int launch_apf_update(float* ema, float* ema_abs, const float* delta, float* score, long long n, float alpha,
                      cudaStream_t s);

// ---- LLaMA glue (K7)
int launch_embedding_fwd(const int* tokens, const __nv_bfloat16* table, __nv_bfloat16* out, int T, int h,
                         cudaStream_t s);
int launch_embedding_bwd(const int* tokens, const __nv_bfloat16* dout, float* gtable, int T, int h, cudaStream_t s);
int launch_rmsnorm_fwd(const __nv_bfloat16* x, const __nv_bfloat16* g, __nv_bfloat16* y, float* rstd, int T, int h,
                       float eps, cudaStream_t s);
// dx = residual + rmsnorm_bwd(dy); dg += sum_t dy * x * rstd
int launch_rmsnorm_bwd(const __nv_bfloat16* x, const __nv_bfloat16* g, const float* rstd, const __nv_bfloat16* dy,
                       const __nv_bfloat16* residual, __nv_bfloat16* dx, float* dg, int T, int h, cudaStream_t s);
int launch_rope_fwd(__nv_bfloat16* qkv, const float2* cs, int T, int seq, int nh, int nkv, int hd, cudaStream_t s);
// K7 attention (flash_attn.cu): tcgen05 flash attention over the packed qkv [B*S, (nh + 2 nkv) hd]
// (after RoPE), S % 128 == 0, hd in {64, 128}, native GQA. Forward: out [B*S, nh*hd] (row stride
// ldo), lse [B, nh, S] (log2 domain). Backward: dout [B*S, nh*hd] contiguous; D [B, nh, S] and
// dq_acc [B*S, nh*hd] fp32 are scratch; dq|dk|dv are written packed into dqkv (may be qkv itself),
// with the RoPE backward on dq and dk when rope ((cos, sin) [S][hd/2]) is not null.
int launch_flash_attn_fwd(const __nv_bfloat16* qkv, __nv_bfloat16* out, long long ldo, float* lse, int B, int S,
                          int nh, int nkv, int hd, float scale, bool causal, cudaStream_t s);
// development aid (PF_ATTN_PROF=1): per-role cycle counters of the first CTA, copied out and reset
int flash_attn_prof_read(unsigned long long* out32);
int launch_flash_attn_bwd(const __nv_bfloat16* qkv, const __nv_bfloat16* out, const __nv_bfloat16* dout,
                          const float* lse, float* D, float* dq_acc, __nv_bfloat16* dqkv, const float2* rope, int B,
                          int S, int nh, int nkv, int hd, float scale, bool causal, cudaStream_t s);
int launch_swiglu_fwd(const __nv_bfloat16* gu, __nv_bfloat16* a, int T, int ffn, cudaStream_t s);
int launch_swiglu_bwd(const __nv_bfloat16* gu, const __nv_bfloat16* da, __nv_bfloat16* dgu, int T, int ffn,
                      cudaStream_t s);
// in place: logits -> dlogits = (softmax - onehot) * grad_scale; loss_sum += sum_t (lse - x_target) * loss_scale
int launch_cross_entropy(__nv_bfloat16* logits, const int* targets, float* loss_sum, int T, int V, float grad_scale,
                         float loss_scale, cudaStream_t s);
int launch_init_normal(float* master, __nv_bfloat16* weights, long long n, float stddev, uint64_t seed,
                       cudaStream_t s);
int launch_fill(float* master, __nv_bfloat16* weights, long long n, float value, cudaStream_t s);
int launch_rope_table(float2* cs, int seq, int hd, float theta, cudaStream_t s);
int launch_random_tokens(int* tokens, long long n, int vocab, uint64_t seed, cudaStream_t s);

}  // namespace pf
