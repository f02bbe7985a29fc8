// ViT encoder stage (ViT-L/32, 224^2 images, 32^2 patches -> 49 + cls
// = 50 tokens, 64 images per microbatch -> T = 3200, GPipe PP4 M8).
//
// Pre-LN encoder layer: h1 = LN1(x); qkv = h1 Wqkv^T + bqkv; bidirectional attention;
// x2 = x + attn Wo^T + bo; h2 = LN2(x2); x' = x2 + GELU(h2 W1^T + b1) W2^T + b2.
// First stage: patch embedding (a freezable [h, 3*32*32] matrix) + cls + positions.
// Last stage: LN on the cls rows, classification head (freezable [classes, h]) + CE.
// The freeze units, masked dW (K3), K5 lists, optimizer and split backward are the
// shared Stage machinery; weight matrices are freezable, biases / LN / embeddings dense.
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "stage.hpp"
#include "stage_ops.hpp"
#include "vit_kernels.cuh"
#include <string>
#include <cstdlib>

namespace pf {

namespace {

#define PF_TRY(expr)              \
  do {                            \
    const int _rc = (expr);       \
    if (_rc != PF_OK) return _rc; \
  } while (0)
#define PF_CUDA(expr)                              \
  do {                                             \
    if ((expr) != cudaSuccess) return PF_ERR_CUDA; \
  } while (0)

using namespace ops;

struct VitLayerParams {
  ParamSlice wqkv, wo, w1, w2;                           // freezable
  ParamSlice bqkv, bo, b1, b2, ln1g, ln1b, ln2g, ln2b;   // dense
};

struct VitSavedLayer {
  __nv_bfloat16 *x = nullptr, *h1 = nullptr, *qkv = nullptr, *x2 = nullptr, *h2 = nullptr, *pre = nullptr,
                *act = nullptr;
  float *mu1 = nullptr, *r1 = nullptr, *mu2 = nullptr, *r2 = nullptr;
  const __nv_bfloat16* attn_out = nullptr;
  long long attn_ld = 0;
  __nv_bfloat16* ao = nullptr;  // attention output [T, h]
  float* lse = nullptr;         // and its row log-sum-exp [B][nh][S]
  __nv_bfloat16 *dy = nullptr, *dx2 = nullptr;  // kept from B to W
  const __nv_bfloat16* dy_w = nullptr;          // the output gradient W reads (dy or the incoming buffer)
};

struct VitSlot {
  std::vector<VitSavedLayer> layers;
  __nv_bfloat16* patches = nullptr;  // first stage: [B*np, patch_dim] input
  __nv_bfloat16* emb = nullptr;      // first stage: patch embeddings, then (split) their gradient
  __nv_bfloat16* x_out = nullptr;
  __nv_bfloat16 *xc = nullptr, *hc = nullptr, *logits = nullptr;  // last stage: cls rows (padded), LN, logits
  float *muc = nullptr, *rc = nullptr;
};

class VitStage final : public Stage {
 public:
  VitStage(const ModelConfig& cfg, const StageSpec& spec, int slots, uint64_t seed, int device, bool split)
      : Stage(cfg, spec, device, split), seed_(seed) {
    const int h = cfg.hidden;
    if (h % 128 || cfg.ffn % 128 || cfg.n_kv_heads != cfg.n_heads || cfg.n_heads * cfg.head_dim != h ||
        cfg.vocab % 8 || cfg.patch_dim() % 64 || cfg.seq != cfg.patches() + 1 ||
        (cfg.micro_batch * cfg.patches()) % 64)
      throw std::invalid_argument("vit stage: unsupported shape");
    B_ = cfg.micro_batch;
    S_ = cfg.seq;
    np_ = S_ - 1;
    T_ = cfg.tokens();
    // short sequences (ViT-L/32: 50 tokens) use the per-(image, head) kernel (vit_attention.cu);
    // sequences of whole 128-token blocks the bidirectional tcgen05 flash attention (flash_attn.cu)
    own_attn_ = S_ <= 64 && cfg.head_dim == 64;
    if (!own_attn_ && (S_ % 128 != 0 || (cfg.head_dim != 64 && cfg.head_dim != 128)))
      throw std::invalid_argument("vit stage: attention needs seq <= 64 with head_dim 64, or seq % 128 == 0");
    Mh_ = (B_ + 127) / 128 * 128;
    const int nl = spec.layer_end - spec.layer_begin;
    layers_.resize(static_cast<std::size_t>(nl));
    if (spec.first) patch_w_ = add_matrix(h, cfg.patch_dim(), true);
    for (auto& L : layers_) {
      L.wqkv = add_matrix(3 * h, h, true);
      L.wo = add_matrix(h, h, true);
      L.w1 = add_matrix(cfg.ffn, h, true);
      L.w2 = add_matrix(h, cfg.ffn, true);
    }
    if (spec.last) head_ = add_matrix(cfg.vocab, h, true);
    end_unit_matrices();
    for (auto& L : layers_) {
      L.bqkv = add_dense(3 * h);
      L.bo = add_dense(h);
      L.b1 = add_dense(cfg.ffn);
      L.b2 = add_dense(h);
      L.ln1g = add_dense(h);
      L.ln1b = add_dense(h);
      L.ln2g = add_dense(h);
      L.ln2b = add_dense(h);
    }
    if (spec.first) {
      patch_b_ = add_dense(h);
      cls_ = add_dense(h);
      pos_ = add_dense(static_cast<long long>(S_) * h);
    }
    if (spec.last) {
      lnfg_ = add_dense(h);
      lnfb_ = add_dense(h);
      headb_ = add_dense(cfg.vocab);
    }
    allocate_parameters(seed);
    // dense init: LN gains 1, biases 0, cls / positions N(0, init_std)
    auto fill = [&](const ParamSlice& p, float v) { launch_fill(master_ + p.offset, weights_ + p.offset, p.count, v, nullptr); };
    for (auto& L : layers_) {
      for (const ParamSlice* p : {&L.bqkv, &L.bo, &L.b1, &L.b2, &L.ln1b, &L.ln2b}) fill(*p, 0.f);
      fill(L.ln1g, 1.f);
      fill(L.ln2g, 1.f);
    }
    if (spec.first) {
      fill(patch_b_, 0.f);
      launch_init_normal(master_ + cls_.offset, weights_ + cls_.offset, cls_.count,
                         cfg.init_std, seed * 7919ULL + 23ULL, nullptr);
      launch_init_normal(master_ + pos_.offset, weights_ + pos_.offset, pos_.count, cfg.init_std,
                         seed * 7919ULL + 29ULL, nullptr);
    }
    if (spec.last) {
      fill(lnfg_, 1.f);
      fill(lnfb_, 0.f);
      fill(headb_, 0.f);
    }

    const long long T = T_;
    slots_.resize(static_cast<std::size_t>(slots));
    for (auto& sl : slots_) {
      sl.layers.resize(static_cast<std::size_t>(nl));
      for (auto& L : sl.layers) {
        L.x = alloc_bf16(T * h);
        L.h1 = alloc_bf16(T * h);
        L.qkv = alloc_bf16(T * 3 * h);
        L.x2 = alloc_bf16(T * h);
        L.h2 = alloc_bf16(T * h);
        L.pre = alloc_bf16(T * cfg.ffn);
        L.act = alloc_bf16(T * cfg.ffn);
        L.mu1 = alloc_f32(T);
        L.r1 = alloc_f32(T);
        L.mu2 = alloc_f32(T);
        L.r2 = alloc_f32(T);
        L.ao = alloc_bf16(T * h);
        L.lse = alloc_f32(static_cast<long long>(B_) * cfg.n_heads * S_);
        L.dy = alloc_bf16(T * h);
        L.dx2 = alloc_bf16(T * h);
      }
      sl.x_out = alloc_bf16(T * h);
      if (spec.first) {
        sl.patches = alloc_bf16(static_cast<long long>(B_) * np_ * cfg.patch_dim());
        sl.emb = alloc_bf16(static_cast<long long>(B_) * np_ * h);
      }
      if (spec.last) {
        sl.xc = alloc_bf16(static_cast<long long>(Mh_) * h);
        sl.hc = alloc_bf16(static_cast<long long>(Mh_) * h);
        sl.logits = alloc_bf16(static_cast<long long>(Mh_) * cfg.vocab);
        sl.muc = alloc_f32(Mh_);
        sl.rc = alloc_f32(Mh_);
        cudaMemset(sl.hc, 0, static_cast<size_t>(Mh_) * h * 2);  // padding rows stay zero
      }
    }
    d_act_ = alloc_bf16(T * cfg.ffn);
    d_h_ = alloc_bf16(T * h);
    d_attn_ = alloc_bf16(T * h);
    if (!own_attn_) {
      attn_D_ = alloc_f32(static_cast<long long>(B_) * cfg.n_heads * S_);
      dq_acc_ = alloc_f32(T * h);
    }
    d_y_ = alloc_bf16(T * h);
    d_tmp_ = alloc_bf16(T * h);
    if (spec.last) {
      d_hc_ = alloc_bf16(static_cast<long long>(Mh_) * h);
      d_xc_ = alloc_bf16(static_cast<long long>(Mh_) * h);
    }
    if (cudaDeviceSynchronize() != cudaSuccess) throw std::runtime_error("vit stage: initialisation failed");
  }

  ~VitStage() override { cudaSetDevice(device_); }

  const __nv_bfloat16* output(int slot) const override { return slots_[static_cast<std::size_t>(slot)].x_out; }

  int forward(int slot, int microbatch, const int* /*tokens*/, const int* targets, const __nv_bfloat16* x_in,
              float* loss_sum, cudaStream_t s) override {
    if (slot < 0 || slot >= static_cast<int>(slots_.size())) return PF_ERR_INVALID;
    VitSlot& sl = slots_[static_cast<std::size_t>(slot)];
    const int h = cfg_.hidden, ffn = cfg_.ffn, pd = cfg_.patch_dim(), Tp = B_ * np_;
    const int nl = static_cast<int>(layers_.size());
    __nv_bfloat16* x0 = nl > 0 ? sl.layers[0].x : sl.x_out;
    if (spec_.first) {  // synthetic images of this microbatch -> patch embeddings -> tokens
      PF_TRY(launch_synthetic_patches(sl.patches, static_cast<long long>(Tp) * pd,
                                      seed_ * 0x9e3779b97f4a7c15ULL + static_cast<uint64_t>(microbatch), s));
      PF_TRY(gemm_fwd(sl.patches, pd, w(patch_w_), pd, sl.emb, h, Tp, h, pd, EPI_STORE_BF16, s));
      PF_TRY(launch_vit_embed_fwd(sl.emb, w(patch_b_), w(cls_), w(pos_), x0, B_, S_, h, s));
    } else {
      if (!x_in) return PF_ERR_INVALID;
      PF_CUDA(cudaMemcpyAsync(x0, x_in, static_cast<size_t>(T_) * h * 2, cudaMemcpyDeviceToDevice, s));
    }
    const float scale = 1.0f / std::sqrt(static_cast<float>(cfg_.head_dim));
    for (int li = 0; li < nl; ++li) {
      VitSavedLayer& L = sl.layers[static_cast<std::size_t>(li)];
      const VitLayerParams& P = layers_[static_cast<std::size_t>(li)];
      PF_TRY(launch_layernorm_fwd(L.x, w(P.ln1g), w(P.ln1b), L.h1, L.mu1, L.r1, T_, h, cfg_.norm_eps, s));
      PF_TRY(gemm_fwd_bias(L.h1, h, w(P.wqkv), h, L.qkv, 3LL * h, w(P.bqkv), T_, 3 * h, h, s));
      if (own_attn_) {
        PF_TRY(launch_vit_attn_fwd(L.qkv, L.ao, L.lse, B_, S_, cfg_.n_heads, cfg_.head_dim, scale, s));
        L.attn_out = L.ao;
        L.attn_ld = h;
      } else {
        PF_TRY(launch_flash_attn_fwd(L.qkv, L.ao, h, L.lse, B_, S_, cfg_.n_heads, cfg_.n_heads, cfg_.head_dim, scale,
                                     false, s));
        L.attn_out = L.ao;
        L.attn_ld = h;
      }
      PF_TRY(gemm_fwd_resid_bias(L.attn_out, L.attn_ld, w(P.wo), h, L.x2, L.x, h, w(P.bo), T_, h, h, s));
      PF_TRY(launch_layernorm_fwd(L.x2, w(P.ln2g), w(P.ln2b), L.h2, L.mu2, L.r2, T_, h, cfg_.norm_eps, s));
      // MLP up-projection with bias and GELU fused in the epilogue; the bench.py roofline probe
      // brackets that launch (or, unfused, the GEMM without the GELU kernel)
      const bool probe = probe_kind() == PROBE_GATE_UP_GEMM;
      if (probe && !fuse_swiglu()) {
        probe_begin(s);
        PF_TRY(gemm_fwd_bias(L.h2, h, w(P.w1), h, L.pre, ffn, w(P.b1), T_, ffn, h, s));
        probe_end(s);
        PF_TRY(launch_gelu_fwd(L.pre, L.act, static_cast<long long>(T_) * ffn, s));
      } else {
        if (probe) probe_begin(s);
        PF_TRY(gemm_fwd_bias_gelu(L.h2, h, w(P.w1), h, w(P.b1), L.pre, L.act, T_, ffn, h, s));
        if (probe) probe_end(s);
      }
      __nv_bfloat16* next = li + 1 < nl ? sl.layers[static_cast<std::size_t>(li + 1)].x : sl.x_out;
      PF_TRY(gemm_fwd_resid_bias(L.act, ffn, w(P.w2), ffn, next, L.x2, h, w(P.b2), T_, h, ffn, s));
    }
    if (spec_.last) {  // head on the cls rows; mean CE over the microbatch's images
      if (!targets || !loss_sum) return PF_ERR_INVALID;
      PF_TRY(launch_gather_rows(sl.x_out, sl.xc, B_, S_, h, s));
      PF_TRY(launch_layernorm_fwd(sl.xc, w(lnfg_), w(lnfb_), sl.hc, sl.muc, sl.rc, B_, h, cfg_.norm_eps, s));
      PF_TRY(gemm_fwd(sl.hc, h, w(head_), h, sl.logits, cfg_.vocab, Mh_, cfg_.vocab, h, EPI_STORE_BF16, s));
      PF_TRY(launch_add_bias(sl.logits, cfg_.vocab, w(headb_), B_, cfg_.vocab, s));
      PF_TRY(launch_cross_entropy(sl.logits, targets, loss_sum, B_, cfg_.vocab, 1.0f / B_, 1.0f / B_, s));
    }
    return PF_OK;
  }

  int backward(int slot, const int* /*tokens*/, const uint64_t* frozen_words, const __nv_bfloat16* dy,
               __nv_bfloat16* dx_out, int stamp, cudaStream_t s) override {
    if (slot < 0 || slot >= static_cast<int>(slots_.size()) || (!frozen_words && !split_)) return PF_ERR_INVALID;
    VitSlot& sl = slots_[static_cast<std::size_t>(slot)];
    const int h = cfg_.hidden, ffn = cfg_.ffn;
    const int nl = static_cast<int>(layers_.size());
    if (!split_) PF_TRY(build_unit_lists(frozen_words, s));
    __nv_bfloat16* top = nl > 0 ? sl.layers[static_cast<std::size_t>(nl - 1)].dy : d_y_;
    const __nv_bfloat16* dcur = dy;
    if (spec_.last) {
      PF_TRY(launch_bias_grad(sl.logits, cfg_.vocab, g(headb_), B_, cfg_.vocab, s));
      PF_TRY(gemm_dx(sl.logits, cfg_.vocab, w(head_), h, d_hc_, h, Mh_, h, cfg_.vocab, EPI_STORE_BF16, s));
      PF_TRY(launch_layernorm_bwd(sl.xc, w(lnfg_), sl.muc, sl.rc, d_hc_, nullptr, d_xc_, g(lnfg_), g(lnfb_), nullptr, B_, h,
                                  s));
      PF_TRY(launch_scatter_rows(d_xc_, top, B_, S_, h, s));
      dcur = top;
    } else if (split_ && nl > 0 && dcur) {
      PF_CUDA(cudaMemcpyAsync(top, dcur, static_cast<size_t>(T_) * h * 2, cudaMemcpyDeviceToDevice, s));
      dcur = top;
    }
    if (!dcur) return PF_ERR_INVALID;
    const float scale = 1.0f / std::sqrt(static_cast<float>(cfg_.head_dim));
    for (int li = nl - 1; li >= 0; --li) {
      VitSavedLayer& L = sl.layers[static_cast<std::size_t>(li)];
      const VitLayerParams& P = layers_[static_cast<std::size_t>(li)];
      L.dy_w = dcur;
      __nv_bfloat16* dpre = L.pre;  // pre is dead once GELU' is applied
      __nv_bfloat16* dx2 = L.dx2;
      __nv_bfloat16* dqkv = L.qkv;  // qkv is dead after the attention backward
      // MLP
      // b2's gradient: the column sums of this layer's output gradient (the layer above's
      // LayerNorm-1 backward produced them in the same pass, except for the top layer)
      if (li == nl - 1) PF_TRY(launch_bias_grad(dcur, h, g(P.b2), T_, h, s));
      // fc2 dX with GELU' and b1's gradient (column sums of dpre) in the epilogue
      PF_TRY(gemm_dx_dgelu(dcur, h, w(P.w2), ffn, L.pre, d_act_, dpre, g(P.b1), T_, ffn, h, s));
      PF_TRY(gemm_dx(dpre, ffn, w(P.w1), h, d_h_, h, T_, h, ffn, EPI_STORE_BF16, s));
      // LayerNorm-2 backward; bo's gradient (column sums of dx2) in the same pass
      PF_TRY(launch_layernorm_bwd(L.x2, w(P.ln2g), L.mu2, L.r2, d_h_, dcur, dx2, g(P.ln2g), g(P.ln2b), g(P.bo), T_, h,
                                  s));
      // attention
      PF_TRY(gemm_dx(dx2, h, w(P.wo), h, d_attn_, h, T_, h, h, EPI_STORE_BF16, s));
      if (own_attn_) {  // dq|dk|dv straight into the packed dqkv (over qkv), bqkv's gradient alongside
        PF_TRY(launch_vit_attn_bwd(L.qkv, L.ao, d_attn_, L.lse, dqkv, g(P.bqkv), B_, S_, cfg_.n_heads,
                                   cfg_.head_dim, scale, s));
      } else {  // no RoPE in the ViT: dq|dk|dv packed over qkv as they are
        PF_TRY(launch_flash_attn_bwd(L.qkv, L.ao, d_attn_, L.lse, attn_D_, dq_acc_, dqkv, nullptr, B_, S_,
                                     cfg_.n_heads, cfg_.n_heads, cfg_.head_dim, scale, false, s));
      }
      if (!own_attn_) PF_TRY(launch_bias_grad(dqkv, 3LL * h, g(P.bqkv), T_, 3 * h, s));
      PF_TRY(gemm_dx(dqkv, 3LL * h, w(P.wqkv), h, d_h_, h, T_, h, 3 * h, EPI_STORE_BF16, s));
      __nv_bfloat16* out;
      if (li > 0) out = sl.layers[static_cast<std::size_t>(li - 1)].dy;
      else out = spec_.first ? d_tmp_ : dx_out;
      if (!out) return PF_ERR_INVALID;
      // LayerNorm-1 backward; its output is the layer below's output gradient, whose column sums
      // are that layer's b2 gradient
      float* b2_below = li > 0 ? g(layers_[static_cast<std::size_t>(li - 1)].b2) : nullptr;
      PF_TRY(launch_layernorm_bwd(L.x, w(P.ln1g), L.mu1, L.r1, d_h_, dx2, out, g(P.ln1g), g(P.ln1b), b2_below, T_, h,
                                  s));
      dcur = out;
    }
    if (spec_.first) {
      // patch embeddings are dead after the forward: their gradient overwrites them
      PF_TRY(launch_vit_embed_bwd(dcur, sl.emb, g(pos_), g(cls_), g(patch_b_), B_, S_, h, s));
    } else if (nl == 0 && dx_out && dcur != dx_out) {
      PF_CUDA(cudaMemcpyAsync(dx_out, dcur, static_cast<size_t>(T_) * h * 2, cudaMemcpyDeviceToDevice, s));
    }
    // K3: all masked weight gradients of the microbatch in one launch (split: in W)
    if (!split_) PF_TRY(weight_grads(sl, stamp, s));
    return PF_OK;
  }

  int backward_weight(int slot, const uint64_t* frozen_words, int stamp, cudaStream_t s) override {
    if (!split_ || slot < 0 || slot >= static_cast<int>(slots_.size()) || !frozen_words) return PF_ERR_INVALID;
    PF_TRY(build_unit_lists(frozen_words, s));
    return weight_grads(slots_[static_cast<std::size_t>(slot)], stamp, s);
  }

 private:
  const __nv_bfloat16* w(const ParamSlice& p) const { return weights_ + p.offset; }
  float* g(const ParamSlice& p) const { return grad_ + p.offset; }

  // W: every masked weight gradient of the microbatch in `sl` in one K3 launch
  int weight_grads(VitSlot& sl, int stamp, cudaStream_t s) {
    const int h = cfg_.hidden, ffn = cfg_.ffn;
    std::vector<DwGemm> items;
    items.reserve(4 * layers_.size() + 2);
    if (spec_.last) items.push_back(dw_item(head_, sl.logits, cfg_.vocab, sl.hc, h, B_));
    for (int li = static_cast<int>(layers_.size()) - 1; li >= 0; --li) {
      const VitSavedLayer& L = sl.layers[static_cast<std::size_t>(li)];
      const VitLayerParams& P = layers_[static_cast<std::size_t>(li)];
      items.push_back(dw_item(P.w2, L.dy_w, h, L.act, ffn, T_));
      items.push_back(dw_item(P.w1, L.pre, ffn, L.h2, h, T_));
      items.push_back(dw_item(P.wo, L.dx2, h, L.attn_out, L.attn_ld, T_));
      items.push_back(dw_item(P.wqkv, L.qkv, 3LL * h, L.h1, h, T_));
    }
    if (spec_.first) items.push_back(dw_item(patch_w_, sl.emb, h, sl.patches, cfg_.patch_dim(), B_ * np_));
    PF_TRY(run_dw(items, stamp, s));
    return PF_OK;
  }

  uint64_t seed_;
  int B_ = 0, S_ = 0, np_ = 0, T_ = 0, Mh_ = 0;
  bool own_attn_ = false;
  std::vector<VitLayerParams> layers_;
  ParamSlice patch_w_, patch_b_, cls_, pos_, head_, headb_, lnfg_, lnfb_;
  float* attn_D_ = nullptr;  // flash attention backward scratch (seq % 128 == 0 shapes)
  float* dq_acc_ = nullptr;
  std::vector<VitSlot> slots_;
  __nv_bfloat16 *d_act_ = nullptr, *d_h_ = nullptr, *d_attn_ = nullptr, *d_y_ = nullptr, *d_tmp_ = nullptr,
                *d_hc_ = nullptr,
                *d_xc_ = nullptr;
};

}  // namespace

std::unique_ptr<Stage> make_vit_stage(const ModelConfig& cfg, const StageSpec& spec, int slots, uint64_t seed,
                                      int device, bool split_backward) {
  return std::make_unique<VitStage>(cfg, spec, slots, seed, device, split_backward);
}

}  // namespace pf
