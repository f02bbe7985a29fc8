// One pipeline stage of a LLaMA-shaped decoder on one GPU: parameters,
// per-microbatch saved activations, forward / backward with the masked
// weight-gradient GEMM, and the masked optimizer step.
//
// The reference has no model; its stage step is the pair of CPU stand-ins
// sample_execution (duration, proj/src/timing.cpp:58-65) and run_masked_sgd
// (numerics, proj/src/sandbox.cpp:191-257). Here:
//   forward(m)   f(m,s): K1 GEMMs + glue; w_f is its device time
//   backward(m)  b(m,s): K2 dX GEMMs (w_min part) + K3 dW GEMMs over the
//                unfrozen 128x128 units of mask U_{m,s} (the (1-r) w_param part)
//   optimizer    theta -= (eta/M) * sum_m U_m . g_m  (sandbox.cpp:221,250),
//                units frozen in every microbatch are skipped.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <cstdlib>
#include <vector>

#include "kernels.cuh"
#include "pf_device_internal.hpp"

namespace pf {

struct ModelConfig {
  int hidden = 256;
  int ffn = 1024;
  int n_heads = 4;
  int n_kv_heads = 4;
  int head_dim = 64;
  int vocab = 1024;
  int layers = 8;
  int seq = 128;
  int micro_batch = 4;
  float rope_theta = 500000.f;
  float norm_eps = 1e-5f;
  float init_std = 0.02f;
  // 0: LLaMA decoder (vocab = vocabulary). 1: ViT encoder: seq = patches + 1 (cls),
  // vocab = classes, image / patch / channels give the patch-embedding input width.
  int family = 0;
  int image = 224, patch = 32, channels = 3;

  int tokens() const { return seq * micro_batch; }
  int patch_dim() const { return patch * patch * channels; }
  int patches() const { return (image / patch) * (image / patch); }
  int qkv_dim() const { return (n_heads + 2 * n_kv_heads) * head_dim; }
  int attn_dim() const { return n_heads * head_dim; }
};

struct StageSpec {
  int stage = 1;         // 1-based virtual stage
  int layer_begin = 0;   // [begin, end)
  int layer_end = 0;
  bool first = false;    // embedding lives here
  bool last = false;     // final norm + LM head + loss live here
};

struct ParamSlice {
  long long offset = 0;  // element offset in the flat buffers
  long long count = 0;
  int rows = 0, cols = 0;
  int unit_matrix = -1;  // index into the unit table, -1 for dense params
};

struct LayerParams {
  ParamSlice g1, wqkv, wo, g2, wgu, wd;
};

struct SavedLayer {  // per layer per microbatch slot
  __nv_bfloat16 *x = nullptr, *h1 = nullptr, *qkv = nullptr, *x2 = nullptr, *h2 = nullptr, *gu = nullptr,
                *a = nullptr;
  float *rstd1 = nullptr, *rstd2 = nullptr;
  __nv_bfloat16* ao = nullptr;  // attention output [T, nh*hd] (kept for dWo)
  float* lse = nullptr;         // attention log-sum-exp [B, nh, S] (log2 domain)
  const __nv_bfloat16* attn_out = nullptr;
  long long attn_ld = 0;
  // the layer's output gradient and post-attention residual gradient, kept from B to
  // W (dgu and dqkv are written over gu and qkv); dy_w is the output gradient W reads
  // (dy, or the stage's incoming gradient buffer when W runs inside the same action)
  __nv_bfloat16 *dy = nullptr, *dx2 = nullptr;
  const __nv_bfloat16* dy_w = nullptr;
};

struct Slot {  // one in-flight microbatch
  std::vector<SavedLayer> layers;
  __nv_bfloat16* x_out = nullptr;   // stage output (last layer output / residual stream)
  __nv_bfloat16* hf = nullptr;      // last stage: final norm output
  float* rstdf = nullptr;
  __nv_bfloat16* logits = nullptr;  // last stage: logits -> dlogits in place
  int microbatch = 0;
};

struct OptimCfg {
  int adamw = 0;  // 0: SGD (the reference's optimizer), 1: AdamW
  float lr = 0.f, eps = 1e-8f, weight_decay = 0.f;
  double beta1 = 0.9, beta2 = 0.999;
};

// Shared by every model family: the flat parameter buffers (fp32 master, bf16 copy,
// fp32 gradient), the 128x128 freeze-unit table, the K5p pair lists, the masked K3
// weight-gradient GEMM (CTA pair, every matrix of the microbatch in one launch) and
// the K6 optimizer (with fused K4 APF).
class Stage {
 public:
  virtual ~Stage();
  Stage(const Stage&) = delete;
  Stage& operator=(const Stage&) = delete;

  // x_in: stage input activations [T, h] (ignored on the first stage, which
  // embeds its input). Returns a pointer to the stage output [T, h] inside the slot.
  virtual int forward(int slot, int microbatch, const int* tokens, const int* targets, const __nv_bfloat16* x_in,
                      float* loss_sum, cudaStream_t s) = 0;
  // frozen_words: device bitmask over this stage's units for this microbatch.
  // dy: gradient of the stage output (ignored on the last stage). dx_out
  // receives the gradient of the stage input (ignored on the first stage).
  virtual int backward(int slot, const int* tokens, const uint64_t* frozen_words, const __nv_bfloat16* dy,
                       __nv_bfloat16* dx_out, int stamp, cudaStream_t s) = 0;
  // W of a split backward: the masked weight gradients of the microbatch in `slot`
  // (K5 lists + grouped K3) from the gradients its B left in the slot.
  virtual int backward_weight(int slot, const uint64_t* frozen_words, int stamp, cudaStream_t s) = 0;
  virtual const __nv_bfloat16* output(int slot) const = 0;
  virtual long long matmul_flops_fwd() const;  // 2 * T * (matmul params of the stage)

  bool split_backward() const { return split_; }
  // SGD: theta -= lr * G / M (sandbox.cpp:250). AdamW: g = G / M into per-unit-step AdamW.
  // Units frozen in every microbatch of the step (stamp != this step) are not touched.
  int optimizer_step(const OptimCfg& oc, int microbatches, int stamp, bool apf, float apf_alpha,
                     float apf_threshold, cudaStream_t s);
  int zero_dense_grads(cudaStream_t s);

  int units() const { return total_units_; }
  int words() const { return (total_units_ + 63) / 64; }
  // The next dW (backward / backward_weight) is of a cell with no frozen unit: every matrix runs as
  // whole CTA-pair tiles (gemm_dw_dense) instead of over the K5r lists. Set by the trainer from the
  // host copy of the cell's mask; PF_DW_DENSE=0 turns the fast path off.
  void set_dense_cell(bool dense) { dense_cell_ = dense && dense_allowed(); }
  long long param_count() const { return n_params_; }
  long long unit_param_count() const { return n_unit_params_; }
  const std::vector<UnitMatrix>& unit_matrices() const { return mats_; }
  const ModelConfig& config() const { return cfg_; }
  const StageSpec& spec() const { return spec_; }

  // raw buffers (tests / parity)
  float* master() const { return master_; }
  __nv_bfloat16* weights() const { return weights_; }
  float* grad() const { return grad_; }
  int* unit_stamps() const { return stamps_; }
  int* apf_eligible() const { return apf_eligible_; }
  float* apf_ema() const { return apf_ema_; }
  float* adam_m() const { return adam_m_; }
  float* adam_v() const { return adam_v_; }
  int* unit_steps() const { return unit_steps_; }
  float* apf_ema_abs() const { return apf_ema_abs_; }
  int last_unfrozen_units() const { return last_unfrozen_; }

 protected:
  Stage(const ModelConfig& cfg, const StageSpec& spec, int device, bool split_backward);
  ParamSlice add_matrix(int rows, int cols, bool freezable);
  ParamSlice add_dense(long long n);
  // after the freezable matrices: everything registered later is dense
  void end_unit_matrices() { n_unit_params_ = dense_begin_ = n_params_; }
  // allocate master / weights / grad / stamps / unit lists; matrices ~ N(0, init_std)
  void allocate_parameters(uint64_t seed);
  void* alloc(size_t bytes);
  __nv_bfloat16* alloc_bf16(long long elems) { return static_cast<__nv_bfloat16*>(alloc(static_cast<size_t>(elems) * 2)); }
  float* alloc_f32(long long elems) { return static_cast<float*>(alloc(static_cast<size_t>(elems) * 4)); }
  // K5 (K5p with the CTA-pair dW): this microbatch's unit mask -> per-matrix work lists
  int build_unit_lists(const uint64_t* frozen_words, cudaStream_t s);
  // K3 work item of one matrix: G[w] (+)= dY^T . X over its unfrozen units, K = rows of dY / X
  DwGemm dw_item(const ParamSlice& w, const __nv_bfloat16* dy, long long ldy, const __nv_bfloat16* x,
                 long long ldx, int K) const;
  // K3 over every item in one launch
  int run_dw(const std::vector<DwGemm>& items, int stamp, cudaStream_t s) {
    const int n = static_cast<int>(items.size());
    if (dense_cell_) return gemm_dw_dense(items.data(), n, stamps_, stamp, s);
    switch (dw_kernel_) {
      case DW_ROWPAIRS: return gemm_dw_rowpairs(items.data(), n, stamps_, stamp, s);
      case DW_CTA_PAIRS: return gemm_dw_pairs(items.data(), n, stamps_, stamp, s);
      default: return gemm_dw_units(items.data(), n, stamps_, stamp, s);
    }
  }

  ModelConfig cfg_;
  StageSpec spec_;
  int device_;
  bool split_ = false;
  std::vector<UnitMatrix> mats_;
  UnitMatrix* mats_dev_ = nullptr;
  long long n_params_ = 0, n_unit_params_ = 0, dense_begin_ = 0;
  int total_units_ = 0;
  float* master_ = nullptr;
  __nv_bfloat16* weights_ = nullptr;
  float* grad_ = nullptr;
  int* stamps_ = nullptr;
  float* apf_ema_ = nullptr;
  float* apf_ema_abs_ = nullptr;
  int* apf_eligible_ = nullptr;
  float* adam_m_ = nullptr;
  float* adam_v_ = nullptr;
  int* unit_steps_ = nullptr;
  int dense_steps_ = 0;
  // K3 variant (PF_DW_KERNEL=units|pairs|rows): 1-CTA 128 x 256 tiles over K5r row pairs
  // (default), 1-CTA 128 x 128 units over K5 lists, or CTA-pair 256 x 128 tiles over K5p
  // column pairs (profiles/r1_dw_bench.txt)
  enum DwKernel { DW_UNITS = 0, DW_CTA_PAIRS = 1, DW_ROWPAIRS = 2 };
  int dw_kernel_ = DW_ROWPAIRS;
  int* unit_lists_ = nullptr;  // K5 / K5p / K5r lists
  int* unit_counts_ = nullptr;
  int pair_capacity_ = 0;
  std::vector<void*> allocations_;
  int last_unfrozen_ = 0;
  bool dense_cell_ = false;
  static bool dense_allowed() {  // read per call: tests flip it within one process
    const char* e = std::getenv("PF_DW_DENSE");
    return !(e && e[0] == '0');
  }
};

// LLaMA-shaped decoder stage (RMSNorm, RoPE, GQA causal attention, SwiGLU, LM head).
class LlamaStage final : public Stage {
 public:
  // split_backward: backward() computes only input gradients (B) and keeps what
  // backward_weight() (W) needs in the slot (zbv-split schedules).
  LlamaStage(const ModelConfig& cfg, const StageSpec& spec, int slots, uint64_t seed, int device,
             bool split_backward = false);
  ~LlamaStage() override;

  int forward(int slot, int microbatch, const int* tokens, const int* targets, const __nv_bfloat16* x_in,
              float* loss_sum, cudaStream_t s) override;
  int backward(int slot, const int* tokens, const uint64_t* frozen_words, const __nv_bfloat16* dy,
               __nv_bfloat16* dx_out, int stamp, cudaStream_t s) override;
  int backward_weight(int slot, const uint64_t* frozen_words, int stamp, cudaStream_t s) override;
  const __nv_bfloat16* output(int slot) const override { return slots_[slot].x_out; }

 private:
  // W: every masked weight gradient of the microbatch in `sl` in one K3 launch
  int weight_grads(Slot& sl, int stamp, cudaStream_t s);

  std::vector<LayerParams> layers_;
  ParamSlice emb_, gf_, wlm_;
  float2* rope_ = nullptr;
  std::vector<Slot> slots_;
  // backward workspace
  __nv_bfloat16 *d_a_ = nullptr, *d_h_ = nullptr, *d_attn_ = nullptr, *d_y_ = nullptr, *d_tmp_ = nullptr;
  float* attn_D_ = nullptr;   // attention backward: rowsum(dO * O) [B, nh, S]
  float* dq_acc_ = nullptr;   // attention backward: fp32 dQ accumulator [T, nh*hd]
};

// The stage of `cfg.family` (0 LLaMA decoder, 1 ViT encoder).
std::unique_ptr<Stage> make_stage(const ModelConfig& cfg, const StageSpec& spec, int slots, uint64_t seed,
                                  int device, bool split_backward);

}  // namespace pf
