// extern "C" surface of the stage engine and the memory-bound kernels (include/pf_device.h).
#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>

#include "kernels.cuh"
#include "pf_device_internal.hpp"
#include "vit_kernels.cuh"
#include "pf_device.h"
#include "trainer.hpp"

struct pf_ctx {
  std::unique_ptr<pf::Trainer> trainer;
};

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    const int rc = f();
    if (rc == PF_ERR_CUDA) {
      const cudaError_t e = cudaGetLastError();
      g_err = std::string("cuda: ") + cudaGetErrorString(e);
    }
    return rc;
  } catch (const pipefreeze::config_error& e) {
    g_err = e.what();
    return PF_ERR_CONFIG;
  } catch (const pipefreeze::numerical_error& e) {
    g_err = e.what();
    return PF_ERR_NUMERICAL;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return PF_ERR_DOMAIN;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return PF_ERR_INVALID;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PF_ERR_INTERNAL;
  }
}

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }
const pf::UnitMatrix* U(const pf_unit_matrix* m) { return reinterpret_cast<const pf::UnitMatrix*>(m); }
static_assert(sizeof(pf_unit_matrix) == sizeof(pf::UnitMatrix), "pf_unit_matrix layout");

}  // namespace

extern "C" {

const char* pf_engine_last_error(void) { return g_err.c_str(); }

int pf_mask_to_unit_lists(const uint64_t* words, const pf_unit_matrix* mats, int nmats, int* lists, int* counts,
                          void* stream) {
  return guard([&] { return pf::launch_mask_to_unit_lists(words, U(mats), nmats, lists, counts, S(stream)); });
}

int pf_mask_to_rowpair_lists(const uint64_t* words, const pf_unit_matrix* mats, int nmats, int* lists, int* counts,
                             void* stream) {
  return guard([&] { return pf::launch_mask_to_rowpair_lists(words, U(mats), nmats, lists, counts, S(stream)); });
}

int pf_mask_to_pair_lists(const uint64_t* words, const pf_unit_matrix* mats, int nmats, int* pairs, int* counts,
                          void* stream) {
  return guard([&] { return pf::launch_mask_to_pair_lists(words, U(mats), nmats, pairs, counts, S(stream)); });
}

int pf_masked_sgd_units(float* master, void* weights, const float* grad, const int* stamp_arr, int stamp, float scale,
                        const pf_unit_matrix* mats, int nmats, int total_units, float* ema, float* ema_abs,
                        float apf_alpha, float apf_threshold, int* eligible, void* stream) {
  return guard([&] {
    pf::OptimArgs a{};
    a.master = master;
    a.weights = static_cast<__nv_bfloat16*>(weights);
    a.grad = grad;
    a.unit_stamp = stamp_arr;
    a.stamp = stamp;
    a.scale = scale;
    a.mats = U(mats);
    a.nmats = nmats;
    a.total_units = total_units;
    a.apf_ema = ema;
    a.apf_ema_abs = ema_abs;
    a.apf_alpha = apf_alpha;
    a.apf_threshold = apf_threshold;
    a.apf_eligible = eligible;
    return pf::launch_masked_sgd_units(a, S(stream));
  });
}

int pf_sgd_dense(float* master, void* weights, const float* grad, long long n, float scale, void* stream) {
  return guard([&] {
    return pf::launch_sgd_dense(master, static_cast<__nv_bfloat16*>(weights), grad, n, scale, S(stream));
  });
}

int pf_apf_update(float* ema, float* ema_abs, const float* delta, float* score, long long n, float alpha,
                  void* stream) {
  return guard([&] { return pf::launch_apf_update(ema, ema_abs, delta, score, n, alpha, S(stream)); });
}

int pf_rmsnorm_fwd(const void* x, const void* g, void* y, float* rstd, int T, int h, float eps, void* stream) {
  return guard([&] {
    return pf::launch_rmsnorm_fwd(static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(g),
                                  static_cast<__nv_bfloat16*>(y), rstd, T, h, eps, S(stream));
  });
}

int pf_rmsnorm_bwd(const void* x, const void* g, const float* rstd, const void* dy, const void* residual, void* dx,
                   float* dg, int T, int h, void* stream) {
  return guard([&] {
    return pf::launch_rmsnorm_bwd(static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(g), rstd,
                                  static_cast<const __nv_bfloat16*>(dy), static_cast<const __nv_bfloat16*>(residual),
                                  static_cast<__nv_bfloat16*>(dx), dg, T, h, S(stream));
  });
}

int pf_swiglu_fwd(const void* gu, void* a, int T, int ffn, void* stream) {
  return guard([&] {
    return pf::launch_swiglu_fwd(static_cast<const __nv_bfloat16*>(gu), static_cast<__nv_bfloat16*>(a), T, ffn,
                                 S(stream));
  });
}

int pf_layernorm_fwd(const void* x, const void* g, const void* b, void* y, float* mean, float* rstd, int T, int h,
                     float eps, void* stream) {
  return guard([&] {
    return pf::launch_layernorm_fwd(static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(g),
                                    static_cast<const __nv_bfloat16*>(b), static_cast<__nv_bfloat16*>(y), mean, rstd,
                                    T, h, eps, S(stream));
  });
}

int pf_layernorm_bwd(const void* x, const void* g, const float* mean, const float* rstd, const void* dy,
                     const void* residual, void* dx, float* dg, float* db, float* dsum, int T, int h, void* stream) {
  return guard([&] {
    return pf::launch_layernorm_bwd(static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(g), mean,
                                    rstd, static_cast<const __nv_bfloat16*>(dy),
                                    static_cast<const __nv_bfloat16*>(residual), static_cast<__nv_bfloat16*>(dx), dg,
                                    db, dsum, T, h, S(stream));
  });
}

int pf_gelu_fwd(const void* pre, void* act, long long n, void* stream) {
  return guard([&] {
    return pf::launch_gelu_fwd(static_cast<const __nv_bfloat16*>(pre), static_cast<__nv_bfloat16*>(act), n,
                               S(stream));
  });
}

int pf_gelu_bwd(const void* pre, const void* dact, void* dpre, long long n, void* stream) {
  return guard([&] {
    return pf::launch_gelu_bwd(static_cast<const __nv_bfloat16*>(pre), static_cast<const __nv_bfloat16*>(dact),
                               static_cast<__nv_bfloat16*>(dpre), n, S(stream));
  });
}

int pf_swiglu_bwd(const void* gu, const void* da, void* dgu, int T, int ffn, void* stream) {
  return guard([&] {
    return pf::launch_swiglu_bwd(static_cast<const __nv_bfloat16*>(gu), static_cast<const __nv_bfloat16*>(da),
                                 static_cast<__nv_bfloat16*>(dgu), T, ffn, S(stream));
  });
}

int pf_rope_fwd(void* qkv, int T, int seq, int nh, int nkv, int hd, float theta, void* stream) {
  return guard([&] {
    float2* cs = nullptr;
    if (cudaMallocAsync(&cs, static_cast<size_t>(seq) * (hd / 2) * sizeof(float2), S(stream)) != cudaSuccess)
      return PF_ERR_CUDA;
    int rc = pf::launch_rope_table(cs, seq, hd, theta, S(stream));
    if (rc == PF_OK) rc = pf::launch_rope_fwd(static_cast<__nv_bfloat16*>(qkv), cs, T, seq, nh, nkv, hd, S(stream));
    cudaFreeAsync(cs, S(stream));
    return rc;
  });
}

int pf_gemm_rope(const void* h, long long ldh, const void* Wqkv, long long ldw, void* qkv, int T, int seq, int nh,
                 int nkv, int hd, int K, float theta, void* stream) {
  return guard([&] {
    if (!h || !Wqkv || !qkv || (hd != 64 && hd != 128)) return static_cast<int>(PF_ERR_INVALID);
    float2* cs = nullptr;
    if (cudaMallocAsync(&cs, static_cast<size_t>(seq) * (hd / 2) * sizeof(float2), S(stream)) != cudaSuccess)
      return static_cast<int>(PF_ERR_CUDA);
    int rc = pf::launch_rope_table(cs, seq, hd, theta, S(stream));
    const int N = (nh + 2 * nkv) * hd;
    if (rc == PF_OK) {
      pf::GemmOut out{qkv, N};
      out.rope = cs;
      out.rope_seq = seq;
      out.rope_hd = hd;
      out.rope_cols = (nh + nkv) * hd;
      rc = pf::gemm_bf16_pair(pf::GemmOperand{h, ldh, false}, pf::GemmOperand{Wqkv, ldw, false}, out, T, N, K, 1.0f,
                              pf::EPI_ROPE, S(stream));
    }
    cudaFreeAsync(cs, S(stream));
    return rc;
  });
}

int pf_vit_attn_fwd(const void* qkv, void* out, float* lse, int B, int seq, int nh, int hd, float scale,
                    void* stream) {
  return guard([&] {
    return pf::launch_vit_attn_fwd(static_cast<const __nv_bfloat16*>(qkv), static_cast<__nv_bfloat16*>(out), lse, B,
                                   seq, nh, hd, scale, S(stream));
  });
}

int pf_vit_attn_bwd(const void* qkv, const void* out, const void* dout, const float* lse, void* dqkv, float* dbias,
                    int B, int seq, int nh, int hd, float scale, void* stream) {
  return guard([&] {
    return pf::launch_vit_attn_bwd(static_cast<const __nv_bfloat16*>(qkv), static_cast<const __nv_bfloat16*>(out),
                                   static_cast<const __nv_bfloat16*>(dout), lse, static_cast<__nv_bfloat16*>(dqkv),
                                   dbias, B, seq, nh, hd, scale, S(stream));
  });
}

int pf_flash_attn_fwd(const void* qkv, void* out, float* lse, int B, int seq, int nh, int nkv, int hd, float scale,
                      int causal, void* stream) {
  return guard([&] {
    return pf::launch_flash_attn_fwd(static_cast<const __nv_bfloat16*>(qkv), static_cast<__nv_bfloat16*>(out),
                                     static_cast<long long>(nh) * hd, lse, B, seq, nh, nkv, hd, scale, causal != 0,
                                     S(stream));
  });
}

int pf_flash_attn_prof(unsigned long long* out32) {
  return guard([&] { return pf::flash_attn_prof_read(out32); });
}

int pf_flash_attn_bwd(const void* qkv, const void* out, const void* dout, const float* lse, void* dqkv, int B, int seq,
                      int nh, int nkv, int hd, float scale, int causal, float rope_theta, void* stream) {
  return guard([&] {
    const long long T = static_cast<long long>(B) * seq;
    float* D = nullptr;
    float* acc = nullptr;
    float2* cs = nullptr;
    int rc = PF_OK;
    if (cudaMallocAsync(&D, static_cast<size_t>(T) * nh * 4, S(stream)) != cudaSuccess ||
        cudaMallocAsync(&acc, static_cast<size_t>(T) * nh * hd * 4, S(stream)) != cudaSuccess)
      rc = PF_ERR_CUDA;
    if (rc == PF_OK && rope_theta > 0.f) {
      if (cudaMallocAsync(&cs, static_cast<size_t>(seq) * (hd / 2) * sizeof(float2), S(stream)) != cudaSuccess)
        rc = PF_ERR_CUDA;
      else
        rc = pf::launch_rope_table(cs, seq, hd, rope_theta, S(stream));
    }
    if (rc == PF_OK)
      rc = pf::launch_flash_attn_bwd(static_cast<const __nv_bfloat16*>(qkv), static_cast<const __nv_bfloat16*>(out),
                                     static_cast<const __nv_bfloat16*>(dout), lse, D, acc,
                                     static_cast<__nv_bfloat16*>(dqkv), cs, B, seq, nh, nkv, hd, scale, causal != 0,
                                     S(stream));
    if (D) cudaFreeAsync(D, S(stream));
    if (acc) cudaFreeAsync(acc, S(stream));
    if (cs) cudaFreeAsync(cs, S(stream));
    return rc;
  });
}

int pf_cross_entropy(void* logits, const int* targets, float* loss_sum, int T, int V, float grad_scale,
                     float loss_scale, void* stream) {
  return guard([&] {
    return pf::launch_cross_entropy(static_cast<__nv_bfloat16*>(logits), targets, loss_sum, T, V, grad_scale,
                                    loss_scale, S(stream));
  });
}

int pf_trainer_create(const pf_model_cfg* m, const pf_train_cfg* c, pf_ctx** out) {
  return guard([&] {
    if (!m || !c || !out) return PF_ERR_INVALID;
    pf::ModelConfig mc;
    mc.hidden = m->hidden;
    mc.ffn = m->ffn;
    mc.n_heads = m->n_heads;
    mc.n_kv_heads = m->n_kv_heads;
    mc.head_dim = m->head_dim;
    mc.vocab = m->vocab;
    mc.layers = m->layers;
    mc.seq = m->seq;
    mc.micro_batch = m->micro_batch;
    mc.rope_theta = m->rope_theta;
    mc.norm_eps = m->norm_eps;
    mc.init_std = m->init_std;
    if (m->family < 0 || m->family > 1) return PF_ERR_CONFIG;
    mc.family = m->family;
    if (m->family == 1) {
      mc.image = m->image;
      mc.patch = m->patch;
      mc.channels = m->channels;
      if (mc.patch <= 0 || mc.image % mc.patch || mc.channels <= 0) return PF_ERR_CONFIG;
    }
    pf::TrainConfig tc;
    if (c->kind < 0 || c->kind > 4) return PF_ERR_CONFIG;
    tc.pipeline.schedule_kind = static_cast<pipefreeze::ScheduleKind>(c->kind);
    tc.pipeline.num_ranks = c->ranks;
    tc.pipeline.stages_per_rank = c->stages_per_rank;
    tc.pipeline.num_microbatches = c->microbatches;
    tc.rank = c->rank;
    tc.phases = pipefreeze::PhasePlan{c->phases[0], c->phases[1], c->phases[2], c->phases[3]};
    tc.r_max = c->r_max;
    tc.lr = c->lr;
    tc.seed = c->seed;
    tc.apf = c->apf != 0;
    tc.apf_every = c->apf_every;
    tc.apf_alpha = c->apf_alpha;
    tc.apf_threshold = c->apf_threshold;
    tc.device = c->device;
    tc.mask_threads = c->mask_threads;
    tc.hybrid = c->hybrid != 0;
    tc.hybrid_unit_fraction = c->hybrid_unit_fraction > 0.f ? c->hybrid_unit_fraction : 0.5f;
    if (c->optimizer < 0 || c->optimizer > 1) return PF_ERR_CONFIG;
    tc.optim.adamw = c->optimizer;
    if (c->optimizer == 1) {
      tc.optim.beta1 = c->beta1;
      tc.optim.beta2 = c->beta2;
      tc.optim.eps = c->eps;
      tc.optim.weight_decay = c->weight_decay;
      if (!(c->beta1 >= 0.f && c->beta1 < 1.f && c->beta2 >= 0.f && c->beta2 < 1.f && c->eps > 0.f))
        return PF_ERR_CONFIG;
    }
    if (tc.hybrid && !tc.apf) return PF_ERR_CONFIG;  // hybrid needs the APF metric
    auto ctx = std::make_unique<pf_ctx>();
    ctx->trainer = std::make_unique<pf::Trainer>(mc, tc);
    *out = ctx.release();
    return PF_OK;
  });
}

int pf_trainer_destroy(pf_ctx* ctx) {
  return guard([&] {
    delete ctx;
    return PF_OK;
  });
}

int pf_trainer_step(pf_ctx* ctx, int t, const int32_t* tok, const int32_t* tgt, pf_step_result* out) {
  return pf_trainer_step_masks(ctx, t, tok, tgt, nullptr, out);
}

int pf_trainer_step_masks(pf_ctx* ctx, int t, const int32_t* tok, const int32_t* tgt, const uint64_t* masks,
                          pf_step_result* out) {
  return guard([&] {
    if (!ctx) return PF_ERR_INVALID;
    pf::StepResult r;
    const int rc = ctx->trainer->step(t, tok, tgt, &r, masks);
    if (rc == PF_OK && out) {
      out->loss = r.loss;
      out->batch_ms = r.batch_ms;
      out->optimizer_ms = r.optimizer_ms;
      out->predicted_ms = r.predicted_ms;
      out->mean_ratio = r.mean_ratio;
      out->mask_ms = r.mask_ms;
      out->frozen_units = r.frozen_units;
      out->total_units = r.total_units;
      out->phase = r.phase;
    }
    return rc;
  });
}

int pf_trainer_set_override(pf_ctx* ctx, double ratio) {
  return guard([&] {
    if (!ctx || ratio > 1.0) return PF_ERR_INVALID;
    ctx->trainer->set_override(ratio);
    return PF_OK;
  });
}

int pf_trainer_set_plan(pf_ctx* ctx, const double* ratios) {
  return guard([&] {
    if (!ctx || !ratios) return PF_ERR_INVALID;
    const size_t n = ctx->trainer->plan_ratios().size();
    ctx->trainer->set_plan(std::vector<double>(ratios, ratios + n));
    return PF_OK;
  });
}

int pf_trainer_get_plan(pf_ctx* ctx, double* ratios, double* out3, double* w_min, double* w_max) {
  return guard([&] {
    if (!ctx) return PF_ERR_INVALID;
    auto& tr = *ctx->trainer;
    if (!tr.has_plan()) return PF_ERR_DOMAIN;
    if (ratios) std::copy(tr.plan_ratios().begin(), tr.plan_ratios().end(), ratios);
    if (out3) {
      out3[0] = tr.plan().makespan_base;
      out3[1] = tr.plan().makespan_opt;
      out3[2] = tr.plan().makespan_floor;
    }
    if (w_min || w_max) {
      const auto prof = tr.measured_profile();
      int k = 0;
      for (const auto& [a, b] : prof.all()) {
        if (w_min) w_min[k] = b.w_min;
        if (w_max) w_max[k] = b.w_max;
        ++k;
      }
    }
    return PF_OK;
  });
}

int pf_trainer_action_ms(pf_ctx* ctx, double* ms, int* kinds, int* mbs, int* stages) {
  return guard([&] {
    if (!ctx) return PF_ERR_INVALID;
    const auto& tr = *ctx->trainer;
    for (size_t i = 0; i < tr.actions().size(); ++i) {
      if (ms) ms[i] = i < tr.action_ms().size() ? tr.action_ms()[i] : 0.0;
      if (kinds) kinds[i] = static_cast<int>(tr.actions()[i].kind);  // 0 f, 1 b, 2 w
      if (mbs) mbs[i] = tr.actions()[i].microbatch;
      if (stages) stages[i] = tr.actions()[i].stage;
    }
    return PF_OK;
  });
}

int pf_trainer_get_info(pf_ctx* ctx, pf_trainer_info* info) {
  return guard([&] {
    if (!ctx || !info) return PF_ERR_INVALID;
    auto& tr = *ctx->trainer;
    info->tokens_per_step = tr.tokens_per_step();
    info->params = 0;
    info->unit_params = 0;
    info->matmul_flops_fwd_per_mb = 0;
    for (auto* st : tr.local_stages()) {
      info->params += st->param_count();
      info->unit_params += st->unit_param_count();
      info->matmul_flops_fwd_per_mb += st->matmul_flops_fwd();
    }
    info->units = tr.units_total();
    info->local_stages = static_cast<int>(tr.local_stages().size());
    info->actions = static_cast<int>(tr.actions().size());
    info->lp_solve_ms = tr.lp_solve_ms();
    return PF_OK;
  });
}

int pf_trainer_stage_buffers(pf_ctx* ctx, int i, void** master, void** weights, void** grad, void** stamps,
                             long long* n_params, int* n_units) {
  return guard([&] {
    if (!ctx) return PF_ERR_INVALID;
    auto st = ctx->trainer->local_stages();
    if (i < 0 || i >= static_cast<int>(st.size())) return PF_ERR_INVALID;
    if (master) *master = st[static_cast<size_t>(i)]->master();
    if (weights) *weights = st[static_cast<size_t>(i)]->weights();
    if (grad) *grad = st[static_cast<size_t>(i)]->grad();
    if (stamps) *stamps = st[static_cast<size_t>(i)]->unit_stamps();
    if (n_params) *n_params = st[static_cast<size_t>(i)]->param_count();
    if (n_units) *n_units = st[static_cast<size_t>(i)]->units();
    return PF_OK;
  });
}

int pf_trainer_optim_state(pf_ctx* ctx, int i, void** m, void** v, void** unit_steps) {
  return guard([&] {
    if (!ctx) return PF_ERR_INVALID;
    auto st = ctx->trainer->local_stages();
    if (i < 0 || i >= static_cast<int>(st.size())) return PF_ERR_INVALID;
    if (m) *m = st[static_cast<size_t>(i)]->adam_m();
    if (v) *v = st[static_cast<size_t>(i)]->adam_v();
    if (unit_steps) *unit_steps = st[static_cast<size_t>(i)]->unit_steps();
    return PF_OK;
  });
}

int pf_trainer_last_masks(pf_ctx* ctx, int i, uint64_t* out) {
  return guard([&] {
    if (!ctx || !out) return PF_ERR_INVALID;
    auto st = ctx->trainer->local_stages();
    if (i < 0 || i >= static_cast<int>(st.size())) return PF_ERR_INVALID;
    const int words = st[static_cast<size_t>(i)]->words();
    const int M = ctx->trainer->config().pipeline.num_microbatches;
    const uint64_t* src = ctx->trainer->masks_host(i);
    for (int m = 0; m < M; ++m)
      for (int w = 0; w < words; ++w) out[static_cast<size_t>(m) * words + w] = src[static_cast<size_t>(m) * (words + 1) + w];
    return PF_OK;
  });
}

}  // extern "C"

extern "C" void* pf_trainer_stream(pf_ctx* ctx) { return ctx ? static_cast<void*>(ctx->trainer->stream()) : nullptr; }

#include <nccl.h>

extern "C" int pf_nccl_unique_ids(void* out, int count) {
  return guard([&] {
    if (!out || count <= 0) return PF_ERR_INVALID;
    for (int k = 0; k < count; ++k) {
      ncclUniqueId id;
      if (ncclGetUniqueId(&id) != ncclSuccess) return PF_ERR_NCCL;
      std::memcpy(static_cast<char*>(out) + static_cast<size_t>(k) * sizeof(id), &id, sizeof(id));
    }
    return PF_OK;
  });
}

extern "C" int pf_trainer_apf_base(pf_ctx* ctx, int i, uint64_t* out) {
  return guard([&] {
    if (!ctx || !out) return PF_ERR_INVALID;
    auto st = ctx->trainer->local_stages();
    if (i < 0 || i >= static_cast<int>(st.size())) return PF_ERR_INVALID;
    if (!ctx->trainer->apf_base_ready()) return PF_ERR_DOMAIN;
    const auto base = ctx->trainer->apf_base_mask(i);
    std::copy(base.words().begin(), base.words().end(), out);
    return PF_OK;
  });
}

extern "C" int pf_trainer_action_starts(pf_ctx* ctx, double* start_ms) {
  return guard([&] {
    if (!ctx || !start_ms) return PF_ERR_INVALID;
    const auto& v = ctx->trainer->action_start_ms();
    std::copy(v.begin(), v.end(), start_ms);
    return PF_OK;
  });
}

extern "C" const char* pf_attention_backend(void) {
  return "flash_attn.cu (hand-written tcgen05/TMEM/TMA flash attention, sm_100a)";
}

extern "C" int pf_trainer_comm_ids(pf_ctx* ctx, int* count) {
  return guard([&] {
    if (!ctx || !count) return PF_ERR_INVALID;
    *count = ctx->trainer->comm_ids_needed();
    return PF_OK;
  });
}

extern "C" int pf_trainer_links(pf_ctx* ctx, int* out) {
  return guard([&] {
    if (!ctx || !out) return PF_ERR_INVALID;
    int k = 0;
    for (const auto& l : ctx->trainer->links()) {
      out[k++] = l.kind;
      out[k++] = l.src;
      out[k++] = l.dst;
    }
    return PF_OK;
  });
}

extern "C" int pf_trainer_init_comm(pf_ctx* ctx, const void* ids, int nranks, int rank) {
  return guard([&] { return ctx ? ctx->trainer->init_comm(ids, nranks, rank) : PF_ERR_INVALID; });
}
