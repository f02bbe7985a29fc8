/* pipefreeze device C-ABI (libpf_device.so): hand-written sm_100a kernels and the
 * per-stage training step behind them.
 *
 * The reference (arXiv 2602.05754 `pipefreeze`) has no device layer: its stage
 * step is two CPU stand-ins, the duration model `sample_execution`
 * (proj/src/timing.cpp:58-65) and the masked-SGD numerics `run_masked_sgd`
 * (proj/src/sandbox.cpp:191-257). Each entry point below cites the reference
 * function whose semantics it realises on the device. All pointers are device
 * pointers unless named `host_*`; every call returns a PF_* status (pf_status.h)
 * and is asynchronous on the given stream.
 */
#ifndef PF_DEVICE_H
#define PF_DEVICE_H

#include <stddef.h>
#include <stdint.h>

#include "pf_status.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pf_ctx pf_ctx; /* opaque per-GPU stage context */

/* ------------------------------------------------------------------ kernels */

/* K1/K2/K3: C (op)= alpha * A . B^T with bf16 operands and fp32 TMEM accumulation.
 * A is logical [M,K]; a_mn_major=0: stored row-major [M][lda], 1: stored [K][lda].
 * B is logical [N,K]; b_mn_major=0: stored [N][ldb],       1: stored [K][ldb].
 * epilogue: 0 store bf16, 1 add into bf16 C, 2 fp32 unit-stamped accumulate
 * (requires unit_stamp, block_n=128), 3 store fp32. block_n in {128, 256}, or 512 for the
 * CTA-pair kernel (tcgen05.mma.cta_group::2, 256 x 256 tiles; A K-major; epilogues 0, 1, 3). */
int pf_gemm_bf16(const void* A, int a_mn_major, long long lda, const void* B, int b_mn_major,
                 long long ldb, void* C, long long ldc, int M, int N, int K, float alpha,
                 int epilogue, int block_n, int* unit_stamp, int stamp, void* stream);

/* K3: masked weight gradient G[M,N] += alpha * A . B^T over the 128x128 units
 * listed in unit_list[0..*unit_count) (unit id = row_block * ceil(N/128) + col_block).
 * First touch of a unit in step `stamp` stores, later touches accumulate
 * (G = sum_m U_m . g_m, reference proj/src/sandbox.cpp:232-249). */
int pf_gemm_dw_units(const void* A, int a_mn_major, long long lda, const void* B, int b_mn_major,
                     long long ldb, float* G, long long ldg, int M, int N, int K, float alpha,
                     const int* unit_list, const int* unit_count, int max_units,
                     int* unit_stamp, int stamp_offset, int stamp, void* stream);

/* K3 on a CTA pair (tcgen05.mma.cta_group::2, M = 256 from two units, N = 128): the same
 * masked, unit-stamped G[M,N] (+)= dY^T . X, with dY stored [K][ldy] (logical A [M,K],
 * MN-major) and X stored [K][ldx] (logical B [N,K], MN-major), over the padded pair list
 * pairs[0..*pair_count) that pf_mask_to_pair_lists writes for this matrix (8-byte aligned). */
int pf_gemm_dw_pairs(const void* dY, long long ldy, const void* X, long long ldx, float* G, long long ldg, int M,
                     int N, int K, const int* pairs, const int* pair_count, int* unit_stamp, int stamp_offset,
                     int stamp, void* stream);

/* K3 over ROW PAIRS (default K3 of the stage engine): the same masked, unit-stamped dW, each
 * CTA computing two unfrozen units of one unit row with one 128 x 256 MMA per K step, over the
 * int2 entries {u0, u1 or -1} that pf_mask_to_rowpair_lists writes for this matrix. */
int pf_gemm_dw_rowpairs(const void* dY, long long ldy, const void* X, long long ldx, float* G, long long ldg, int M,
                        int N, int K, const int* entries, const int* entry_count, int* unit_stamp, int stamp_offset,
                        int stamp, void* stream);

/* K3 of a cell with no frozen unit (the stage engine's dense fast path): every unit of the matrix
 * as 256 x 256 CTA-pair tiles (cta_group::2, two unit rows x two unit columns), no work list;
 * same unit-stamp contract (first touch in a step stores, later ones accumulate). */
int pf_gemm_dw_dense(const void* dY, long long ldy, const void* X, long long ldx, float* G, long long ldg, int M,
                     int N, int K, int* unit_stamp, int stamp_offset, int stamp, void* stream);

/* K1 gate|up projection with the SwiGLU activation fused in the CTA-pair epilogue:
 * gu[T, 2*ffn] = h[T, K] . Wgu^T (bf16, Wgu rows interleave 128-blocks [gate b | up b]),
 * a[T, ffn] = silu(gate) * up from the bf16-rounded gu (== pf_swiglu_fwd(gu)). ffn % 128 == 0. */
int pf_gemm_swiglu(const void* h, long long ldh, const void* Wgu, long long ldw, void* gu, void* a, int T, int ffn,
                   int K, void* stream);

/* K2 down-projection backward with the SwiGLU backward fused in the CTA-pair epilogue:
 * d_act = dY[T, K] . Wd[K, ffn] (Wd stored [K][ffn], read MN-major), rounded to bf16, then
 * dgu = swiglu_bwd(gu, d_act) in the interleaved gate|up layout (== pf_swiglu_bwd). */
int pf_gemm_dswiglu(const void* dY, long long ldy, const void* Wd, long long ldw, const void* gu, void* dgu, int T,
                    int ffn, int K, void* stream);

/* ViT MLP with GELU (erf form) fused in the CTA-pair epilogue, staged through TMA:
 * pf_gemm_gelu:  pre[T, ffn] = bf16(x[T, K] . W1[ffn, K]^T + bias), act = gelu(pre) (== GEMM with bias
 *                + pf_gelu_fwd); pf_gemm_dgelu: d_act = dY[T, K] . W2[K, ffn] (W2 stored [K][ffn], read
 *                MN-major) rounded to bf16, dpre = d_act * gelu'(pre) (== GEMM + pf_gelu_bwd); dpre may
 *                alias pre. ffn % 32 == 0. */
/* Bidirectional attention for S <= 64 and head_dim 64 (ViT-L/32), one CTA per (image, head):
 * qkv packed [B S, 3 nh 64], out [B S, nh 64], lse fp32 [B][nh][S]; the backward writes dq|dk|dv
 * into a packed dqkv (may alias qkv) and, when dbias != NULL, adds the qkv bias gradient (the column sums
 * of the bf16 dq|dk|dv, fp32 [3 nh 64]) into dbias. */
/* K7 attention of the LLaMA stages (flash_attn.cu; tcgen05 MMAs into TMEM fed by TMA): causal (or
 * bidirectional) multi-head attention with native GQA over the packed qkv [B*S, (nh + 2 nkv) hd] bf16
 * (after RoPE); S % 128 == 0, hd 64 or 128. out [B*S, nh*hd] bf16, lse [B, nh, S] fp32 (log2 domain).
 * The backward writes dq|dk|dv packed into dqkv [B*S, (nh + 2 nkv) hd] (may be qkv itself); with
 * rope_theta > 0 the rotate-half RoPE backward is applied to dq and dk (inputs were rotated). */
int pf_flash_attn_fwd(const void* qkv, void* out, float* lse, int B, int S, int nh, int nkv, int hd, float scale,
                      int causal, void* stream);
int pf_flash_attn_bwd(const void* qkv, const void* out, const void* dout, const float* lse, void* dqkv, int B, int S,
                      int nh, int nkv, int hd, float scale, int causal, float rope_theta, void* stream);
/* Development aid: with PF_ATTN_PROF=1 in the environment the attention kernels accumulate the first
 * CTA's per-role cycle counts (waits, compute) into 32 counters; this copies them out and resets. */
int pf_flash_attn_prof(unsigned long long* out32);
int pf_vit_attn_fwd(const void* qkv, void* out, float* lse, int B, int S, int nh, int hd, float scale, void* stream);
int pf_vit_attn_bwd(const void* qkv, const void* out, const void* dout, const float* lse, void* dqkv, float* dbias,
                    int B, int S, int nh, int hd, float scale, void* stream);
/* LayerNorm over rows of h (ViT): y = (x - mean) * rstd * g + b, mean / rstd fp32 per row saved for the
 * backward; pf_layernorm_bwd: dx = residual (nullable) + LayerNorm backward of dy, dg / db += column sums
 * of dy * xhat / dy, dsum += column sums of the bf16 dx (the upstream linear layer's bias gradient);
 * dg, db, dsum nullable. One pass for h = 256, 512, 1024. */
int pf_layernorm_fwd(const void* x, const void* g, const void* b, void* y, float* mean, float* rstd, int T, int h,
                     float eps, void* stream);
int pf_layernorm_bwd(const void* x, const void* g, const float* mean, const float* rstd, const void* dy,
                     const void* residual, void* dx, float* dg, float* db, float* dsum, int T, int h, void* stream);
int pf_gelu_fwd(const void* pre, void* act, long long n, void* stream);              /* act = gelu(pre), n % 8 == 0 */
int pf_gelu_bwd(const void* pre, const void* dact, void* dpre, long long n, void* stream); /* dpre = dact * gelu'(pre) */
int pf_gemm_gelu(const void* x, long long ldx, const void* W1, long long ldw, const void* bias, void* pre, void* act,
                 int T, int ffn, int K, void* stream);
int pf_gemm_dgelu(const void* dY, long long ldy, const void* W2, long long ldw, const void* pre, void* dpre,
                  float* db, int T, int ffn, int K, void* stream);  /* db (nullable): += column sums of dpre */

/* Stream-K split of the CTA-pair GEMM: 0 off (default), 1 split every tile, 2 data-parallel
 * full waves + the last wave split over all CTA pairs, -1 auto (mode 2 when the last wave would
 * leave > 8% of the CTA pairs idle). */
int pf_gemm_set_streamk(int mode);

int pf_device_sm_count(void);
const char* pf_device_last_error(void);  /* message of the last failed kernel-level call */
const char* pf_engine_last_error(void);  /* message of the last failed engine / K4-K7 call */

/* One freezable weight matrix of a stage (device-side table entry, 32 bytes). */
typedef struct pf_unit_matrix {
  long long elem_offset; /* into the stage's flat parameter buffers */
  int rows, cols;
  int unit_offset;       /* first unit id of the matrix within the stage */
  int tiles_n;           /* ceil(cols / 128) */
  int units;             /* ceil(rows/128) * tiles_n */
  int pair_offset;       /* first int (even) of the matrix's K5p / K5r list: units + max(groups, rows) slots */
} pf_unit_matrix;

/* K5: frozen-unit bitmask (sample_mask bit order, one bit per 128x128 unit, +1
 * pad word) -> per-matrix lists of unfrozen local unit ids (lists[unit_offset..])
 * and counts[matrix]. mats is a DEVICE array of nmats entries. */
int pf_mask_to_unit_lists(const uint64_t* frozen_words, const pf_unit_matrix* mats, int nmats, int* lists,
                          int* counts, void* stream);

/* K5r: the same mask -> per-matrix ROW-PAIR lists for pf_gemm_dw_rowpairs at lists[pair_offset..]:
 * int2 entries {u0, u1} of unfrozen units of one unit row in row-major order, a row with an odd
 * count ending {u, -1}; counts[matrix] = entries. */
int pf_mask_to_rowpair_lists(const uint64_t* frozen_words, const pf_unit_matrix* mats, int nmats, int* lists,
                             int* counts, void* stream);

/* K5p: the same mask -> per-matrix PAIR lists for pf_gemm_dw_pairs at pairs[pair_offset..]:
 * unit rows cut into bands of 32 (more when a matrix has > 2048 band x column groups),
 * groups (band, column) band by band, each group's unfrozen unit ids top to bottom,
 * padded to an even count with -1; counts[matrix] = padded entry count. */
int pf_mask_to_pair_lists(const uint64_t* frozen_words, const pf_unit_matrix* mats, int nmats, int* pairs,
                          int* counts, void* stream);

/* K6 (+ fused K4): theta -= scale * G over units whose stamp == `stamp`
 * (reference masked update proj/src/sandbox.cpp:221,250). When ema != NULL the
 * APF state of every unit is advanced with delta = -scale*G (0 for untouched
 * units) and eligible[u] counts elements with score < apf_threshold. */
int pf_masked_sgd_units(float* master, void* weights_bf16, const float* grad, const int* unit_stamp, int stamp,
                        float scale, const pf_unit_matrix* mats, int nmats, int total_units, float* ema,
                        float* ema_abs, float apf_alpha, float apf_threshold, int* eligible, void* stream);
int pf_sgd_dense(float* master, void* weights_bf16, const float* grad, long long n, float scale, void* stream);

/* K4: apf_update (reference proj/src/freezectl.cpp:147-156) in fp32 on the device. */
int pf_apf_update(float* ema, float* ema_abs, const float* delta, float* score, long long n, float alpha,
                  void* stream);

/* K7 glue (bf16 activations, fp32 statistics) */
int pf_rmsnorm_fwd(const void* x, const void* g, void* y, float* rstd, int T, int h, float eps, void* stream);
int pf_rmsnorm_bwd(const void* x, const void* g, const float* rstd, const void* dy, const void* residual, void* dx,
                   float* dg, int T, int h, void* stream);
/* gu rows hold gate|up interleaved in 128-blocks: gate j at column (j/128)*256 + j%128, up j 128 later. */
int pf_swiglu_fwd(const void* gu, void* a, int T, int ffn, void* stream);
int pf_swiglu_bwd(const void* gu, const void* da, void* dgu, int T, int ffn, void* stream);
int pf_rope_fwd(void* qkv, int T, int seq, int nh, int nkv, int hd, float theta, void* stream);
/* qkv[T, (nh + 2 nkv) hd] = h[T, K] . Wqkv^T with the rotate-half RoPE of the q and k heads fused in
 * the CTA-pair epilogue (== pf_gemm_bf16 then pf_rope_fwd, bit for bit); hd == 64 or 128. */
int pf_gemm_rope(const void* h, long long ldh, const void* Wqkv, long long ldw, void* qkv, int T, int seq, int nh,
                 int nkv, int hd, int K, float theta, void* stream);
int pf_cross_entropy(void* logits, const int* targets, float* loss_sum, int T, int V, float grad_scale,
                     float loss_scale, void* stream);

/* ------------------------------------------------------------ stage step engine */

typedef struct pf_model_cfg {
  int hidden, ffn, n_heads, n_kv_heads, head_dim, vocab, layers, seq, micro_batch;
  float rope_theta, norm_eps, init_std;
  /* family 0: LLaMA decoder (vocab = vocabulary). family 1: ViT encoder (SURVEY config C5):
   * vocab = classes, seq = (image/patch)^2 + 1, micro_batch = images; synthetic pixels. */
  int family, image, patch, channels;
} pf_model_cfg;

typedef struct pf_train_cfg {
  int kind;             /* 0 gpipe, 1 1f1b, 2 interleaved-1f1b, 3 zbv, 4 zbv-split (B = dX, W = dW actions) */
  int ranks, stages_per_rank, microbatches, rank;
  int phases[4];        /* T_w, T_m, T_f, T_total (PhasePlan) */
  double r_max, lr;
  uint64_t seed;
  int apf, apf_every;
  float apf_alpha, apf_threshold;
  int device, mask_threads;
  int hybrid;                 /* TimelyFreeze + APF masks via reconcile_mask (Alg. 2) */
  float hybrid_unit_fraction; /* unit joins the APF base set when this fraction is eligible */
  int optimizer;              /* 0 SGD (reference sandbox.cpp:250), 1 AdamW (lr above; per-unit bias correction) */
  double beta1, beta2;        /* AdamW only (bias corrections 1 - beta^k are formed in fp64) */
  float eps, weight_decay;
} pf_train_cfg;

typedef struct pf_step_result {
  double loss, batch_ms, optimizer_ms, predicted_ms, mean_ratio, mask_ms;
  long long frozen_units, total_units;
  int phase;
} pf_step_result;

typedef struct pf_trainer_info {
  long long tokens_per_step, params, unit_params, matmul_flops_fwd_per_mb;
  int units, local_stages, actions;
  double lp_solve_ms;
} pf_trainer_info;

/* Alg. 1 driver for this rank: schedule + DAG + controller on the host,
 * Stage engine on the device. */
int pf_trainer_create(const pf_model_cfg* model, const pf_train_cfg* cfg, pf_ctx** out);
int pf_trainer_destroy(pf_ctx* ctx);
/* One training step t (1-based). host_tokens/host_targets: [M][micro_batch*seq]
 * int32 or NULL (device-resident synthetic tokens). */
int pf_trainer_step(pf_ctx* ctx, int t, const int32_t* host_tokens, const int32_t* host_targets,
                    pf_step_result* out);
/* One step with CALLER-OWNED host frozen-unit masks: host_masks holds, per local
 * stage in order, M masks of ceil(units/64) uint64 words in FreezeMask::test bit order
 * (reference proj/include/pipefreeze/freezectl.hpp:41-59: unit u = bit u%64 of word u/64); bits
 * past the last unit are ignored. They replace the controller's masks for this step (no
 * monitoring sample is recorded); the words are copied to HBM before the step's first action.
 * Reference caller: cmd_simulate's run_freezing_masks -> MaskHistory (tools/pipefreeze.cpp:85-171). */
int pf_trainer_step_masks(pf_ctx* ctx, int t, const int32_t* host_tokens, const int32_t* host_targets,
                          const uint64_t* host_masks, pf_step_result* out);
/* ratio < 0: the phase controller + LP plan; ratio in [0,1]: every cell frozen at `ratio`. */
int pf_trainer_set_override(pf_ctx* ctx, double ratio);
int pf_trainer_set_plan(pf_ctx* ctx, const double* ratios /* (s-1)*M + (m-1) */);
/* plan ratios and {base, opt, floor} makespans of the LP on monitored bounds; returns PF_ERR_DOMAIN before T_m.
 * w_min / w_max: one entry per action node in ActionId order (2*S*M, or 3*S*M for zbv-split). */
int pf_trainer_get_plan(pf_ctx* ctx, double* ratios, double* out3, double* w_min, double* w_max);
int pf_trainer_action_ms(pf_ctx* ctx, double* ms, int* kinds, int* microbatches, int* stages);
/* start of each action of the last step relative to the step origin: a CUDA event recorded when
 * pf_trainer_step began enqueueing (ranks that barrier right before the call share one time axis) */
int pf_trainer_action_starts(pf_ctx* ctx, double* start_ms);
int pf_trainer_get_info(pf_ctx* ctx, pf_trainer_info* info);
/* Raw buffers of local stage i (tests): fp32 master / grad, bf16 weights, unit stamps, device unit table. */
int pf_trainer_stage_buffers(pf_ctx* ctx, int local_stage, void** master, void** weights, void** grad,
                             void** stamps, long long* n_params, int* n_units);
/* Multi-rank pipeline: `count` ncclUniqueId blobs (128 B each) created on one rank and
 * shared with all. pf_trainer_init_comm takes pf_trainer_comm_ids() of them: the world
 * communicator (monitoring all-reduce), then one two-rank communicator per P2P link
 * (a cross-rank (activation | gradient, src rank, dst rank) class of DAG rule-3 edges),
 * and must be called on every rank before step 1. */
int pf_nccl_unique_ids(void* out, int count);
int pf_trainer_comm_ids(pf_ctx* ctx, int* count);
/* links[3*k..3*k+2] = (kind 0 act / 1 grad, src rank, dst rank) for k < pf_trainer_comm_ids - 1 */
int pf_trainer_links(pf_ctx* ctx, int* links);
/* The attention implementation of the LLaMA stages (always this library's own flash_attn.cu kernels;
 * ViT stages with seq <= 64 use vit_attention.cu). */
const char* pf_attention_backend(void);
int pf_trainer_init_comm(pf_ctx* ctx, const void* ids, int nranks, int rank);
/* The cudaStream_t the trainer enqueues its step on (for device-side timing by the caller). */
void* pf_trainer_stream(pf_ctx* ctx);
/* Kernels launched by this library so far (all hand-written kernels, not the ATen attention). */
long long pf_device_launch_count(void);
/* In-step kernel probe: while enabled (which = 1: the K1 gate|up GEMM of every layer forward),
 * the stage brackets each launch of that kernel with CUDA events on its own stream.
 * pf_probe_read synchronises, returns the launches seen and their summed duration, and resets. */
int pf_probe_enable(int which);
int pf_probe_read(int* launches, double* total_ms);
/* Hybrid mode: the APF base set of local stage i from the last APF step (ceil(units/64) words);
 * returns PF_ERR_DOMAIN before the first APF step. */
int pf_trainer_apf_base(pf_ctx* ctx, int local_stage, uint64_t* out);
/* The last step's frozen-unit masks of local stage i: M masks of ceil(units/64) words. */
/* AdamW state of a local stage (NULL pointers before the first AdamW step): fp32 m, v
 * (indexed like master) and the per-unit step counts. */
int pf_trainer_optim_state(pf_ctx* ctx, int local_stage, void** m, void** v, void** unit_steps);
int pf_trainer_last_masks(pf_ctx* ctx, int local_stage, uint64_t* out);

#ifdef __cplusplus
}
#endif

#endif
