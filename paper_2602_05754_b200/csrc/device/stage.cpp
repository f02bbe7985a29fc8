#include "stage.hpp"

#include "stage_ops.hpp"
#include "vit_kernels.cuh"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>

namespace pf {

namespace {

constexpr long long kAlign = 64;  // elements: 256 B fp32 / 128 B bf16 (TMA and float4 alignment)

long long round_up(long long v, long long a) { return (v + a - 1) / a * a; }

#define PF_TRY(expr)                \
  do {                              \
    const int _rc = (expr);         \
    if (_rc != PF_OK) return _rc;   \
  } while (0)

#define PF_CUDA(expr)                                      \
  do {                                                     \
    if ((expr) != cudaSuccess) return PF_ERR_CUDA;         \
  } while (0)

}  // namespace

namespace ops {

// CTA-pair (cta_group::2) kernel for the large K1/K2 GEMMs unless PF_GEMM_PAIR=0
bool use_pair() {
  static const bool on = [] {
    const char* e = std::getenv("PF_GEMM_PAIR");
    return !(e && e[0] == '0');
  }();
  return on;
}

// SwiGLU forward/backward in the CTA-pair GEMM epilogues (default), staged through shared
// memory and TMA stores (profiles/r1_swiglu_epilogue.md): at LLaMA-1B shapes forward 0.212 ms
// GEMM + kernel -> 0.188 ms fused, backward 0.144 -> 0.121 ms; LLaMA-8B 0.677 -> 0.636 and
// 0.423 -> 0.371 ms. PF_FUSE_SWIGLU=0 runs GEMM + the standalone kernels.
bool fuse_swiglu() {
  static const bool on = [] {
    const char* e = std::getenv("PF_FUSE_SWIGLU");
    return !(e && e[0] == '0');
  }();
  return on;
}
bool fuse_swiglu_fwd(int /*K*/) { return fuse_swiglu(); }
bool fuse_swiglu_bwd() { return fuse_swiglu(); }

// A GEMM that is one partial wave on the CTA pairs (the ViT-L/32 N = 1024 GEMMs: 52 256 x 256
// tiles on 74 pairs) runs as 128 x 256 tiles of the one-CTA kernel, still one wave (100 tiles on 148
// SMs): 12.4 vs 14.5 us (o dX), 21.7 vs 22.7 (qkv dX), 26.8 vs 28.9 (fc1 dX) back to back,
// profiles/r2_vit_gemm_ab.txt (in the C5 step: 439.8k -> 444.7k and 438.9k -> 438.7k tok/s on two boxes). The o / fc2 forward (bias + residual) stay on the pair kernel: the
// one-CTA kernel's row-per-thread residual reads made the C5 step slower (440.8k -> 428.3k tok/s).
// PF_GEMM_SMALL_ONECTA=0 keeps the pair kernel (A/B).
static bool small_onecta(int M, int N, int epi) {
  static const bool on = [] {
    const char* e = std::getenv("PF_GEMM_SMALL_ONECTA");
    return !(e && e[0] == '0');
  }();
  if (!on || epi != EPI_STORE_BF16) return false;
  const int sms = num_sms();
  const long long pair_tiles = static_cast<long long>((M + 255) / 256) * ((N + 255) / 256);
  const long long cta_tiles = static_cast<long long>((M + 127) / 128) * ((N + 255) / 256);
  return 4 * pair_tiles <= 3 * (sms / 2) && cta_tiles <= sms;
}

int gemm_any(const GemmOperand& A, const GemmOperand& B, void* C, long long ldc, int M, int N, int K, int epi,
             cudaStream_t s) {
  if (use_pair() && M >= 256 && N >= 256 && !small_onecta(M, N, epi))
    return gemm_bf16_pair(A, B, GemmOut{C, ldc}, M, N, K, 1.0f, epi, s);
  return gemm_bf16(A, B, GemmOut{C, ldc}, M, N, K, 1.0f, epi, N >= 256 ? 256 : 128, s);
}

int gemm_fwd(const __nv_bfloat16* A, long long lda, const __nv_bfloat16* W, long long ldw, void* C, long long ldc,
             int M, int N, int K, int epi, cudaStream_t s) {
  // Y[M,N] (+)= A[M,K] . W[N,K]^T, both K-major
  return gemm_any(GemmOperand{A, lda, false}, GemmOperand{W, ldw, false}, C, ldc, M, N, K, epi, s);
}

// Y = R + A . W^T (residual add fused in the epilogue on the CTA-pair kernel)
int gemm_fwd_resid(const __nv_bfloat16* A, long long lda, const __nv_bfloat16* W, long long ldw, __nv_bfloat16* C,
                   const __nv_bfloat16* R, long long ld, int M, int N, int K, cudaStream_t s) {
  if (use_pair() && M >= 256 && N >= 256) {
    GemmOut out{C, ld};
    out.residual = R;
    out.ldr = ld;
    return gemm_bf16_pair(GemmOperand{A, lda, false}, GemmOperand{W, ldw, false}, out, M, N, K, 1.0f, EPI_ADD_BF16,
                          s);
  }
  if (cudaMemcpyAsync(C, R, static_cast<size_t>(M) * ld * 2, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return PF_ERR_CUDA;
  return gemm_bf16(GemmOperand{A, lda, false}, GemmOperand{W, ldw, false}, GemmOut{C, ld}, M, N, K, 1.0f,
                   EPI_ADD_BF16, N >= 256 ? 256 : 128, s);
}

// gu = h . Wgu^T (gate|up interleaved in 128-row blocks) and a = silu(gate) * up; on the
// CTA-pair kernel the activation is computed in the GEMM epilogue from the same tile.
int gemm_fwd_swiglu(const __nv_bfloat16* A, long long lda, const __nv_bfloat16* W, long long ldw, __nv_bfloat16* gu,
                    __nv_bfloat16* a, int M, int ffn, int K, cudaStream_t s) {
  if (use_pair() && fuse_swiglu_fwd(K) && M >= 256 && (2 * ffn) % 256 == 0) {
    GemmOut out{gu, 2LL * ffn};
    out.aux = a;
    out.ldaux = ffn;
    return gemm_bf16_pair(GemmOperand{A, lda, false}, GemmOperand{W, ldw, false}, out, M, 2 * ffn, K, 1.0f,
                          EPI_SWIGLU, s);
  }
  const int rc = gemm_fwd(A, lda, W, ldw, gu, 2LL * ffn, M, 2 * ffn, K, EPI_STORE_BF16, s);
  return rc ? rc : launch_swiglu_fwd(gu, a, M, ffn, s);
}

int gemm_fwd_bias(const __nv_bfloat16* A, long long lda, const __nv_bfloat16* W, long long ldw, __nv_bfloat16* C,
                  long long ldc, const __nv_bfloat16* bias, int M, int N, int K, cudaStream_t s) {
  if (use_pair() && M >= 256 && N >= 256) {
    GemmOut out{C, ldc};
    out.bias = bias;
    return gemm_bf16_pair(GemmOperand{A, lda, false}, GemmOperand{W, ldw, false}, out, M, N, K, 1.0f,
                          EPI_STORE_BF16, s);
  }
  const int rc = gemm_fwd(A, lda, W, ldw, C, ldc, M, N, K, EPI_STORE_BF16, s);
  return rc ? rc : launch_add_bias(C, ldc, bias, M, N, s);
}

int gemm_fwd_resid_bias(const __nv_bfloat16* A, long long lda, const __nv_bfloat16* W, long long ldw,
                        __nv_bfloat16* C, const __nv_bfloat16* R, long long ld, const __nv_bfloat16* bias, int M,
                        int N, int K, cudaStream_t s) {
  if (use_pair() && M >= 256 && N >= 256) {
    GemmOut out{C, ld};
    out.residual = R;
    out.ldr = ld;
    out.bias = bias;
    return gemm_bf16_pair(GemmOperand{A, lda, false}, GemmOperand{W, ldw, false}, out, M, N, K, 1.0f, EPI_ADD_BF16,
                          s);
  }
  const int rc = gemm_fwd_resid(A, lda, W, ldw, C, R, ld, M, N, K, s);
  return rc ? rc : launch_add_bias(C, ld, bias, M, N, s);
}

int gemm_dx(const __nv_bfloat16* dY, long long ldy, const __nv_bfloat16* W, long long ldw, void* C, long long ldc,
            int M, int N, int K, int epi, cudaStream_t s) {
  // dX[M=T, N=in] = dY[T, K=out] . W[out, in]   (W read MN-major, no transpose)
  return gemm_any(GemmOperand{dY, ldy, false}, GemmOperand{W, ldw, true}, C, ldc, M, N, K, epi, s);
}

// d(gate|up) from d(out) = dY . Wd: on the CTA-pair kernel the SwiGLU backward runs in the
// epilogue (d(act) never reaches HBM); otherwise GEMM into d_act then swiglu_bwd.
int gemm_dx_dswiglu(const __nv_bfloat16* dY, long long ldy, const __nv_bfloat16* Wd, long long ldw,
                    const __nv_bfloat16* gu, __nv_bfloat16* d_act, __nv_bfloat16* dgu, int M, int ffn, int K,
                    cudaStream_t s) {
  if (use_pair() && fuse_swiglu_bwd() && M >= 256 && ffn >= 256) {
    GemmOut out{dgu, 2LL * ffn};
    out.residual = gu;
    out.ldr = 2LL * ffn;
    return gemm_bf16_pair(GemmOperand{dY, ldy, false}, GemmOperand{Wd, ldw, true}, out, M, ffn, K, 1.0f,
                          EPI_DSWIGLU, s);
  }
  const int rc = gemm_dx(dY, ldy, Wd, ldw, d_act, ffn, M, ffn, K, EPI_STORE_BF16, s);
  return rc ? rc : launch_swiglu_bwd(gu, d_act, dgu, M, ffn, s);
}

int gemm_fwd_rope(const __nv_bfloat16* A, long long lda, const __nv_bfloat16* W, long long ldw, __nv_bfloat16* qkv,
                  const float2* rope, int M, int seq, int nh, int nkv, int hd, int K, cudaStream_t s) {
  static const bool fuse = [] {
    const char* e = std::getenv("PF_FUSE_ROPE");
    return !(e && e[0] == '0');
  }();
  const int N = (nh + 2 * nkv) * hd;
  if (use_pair() && fuse_swiglu() && fuse && (hd == 64 || hd == 128) && M >= 256 && N % 256 == 0) {
    GemmOut out{qkv, N};
    out.rope = rope;
    out.rope_seq = seq;
    out.rope_hd = hd;
    out.rope_cols = (nh + nkv) * hd;
    return gemm_bf16_pair(GemmOperand{A, lda, false}, GemmOperand{W, ldw, false}, out, M, N, K, 1.0f, EPI_ROPE, s);
  }
  const int rc = gemm_fwd(A, lda, W, ldw, qkv, N, M, N, K, EPI_STORE_BF16, s);
  return rc ? rc : launch_rope_fwd(qkv, rope, M, seq, nh, nkv, hd, s);
}

int gemm_fwd_bias_gelu(const __nv_bfloat16* A, long long lda, const __nv_bfloat16* W, long long ldw,
                       const __nv_bfloat16* bias, __nv_bfloat16* pre, __nv_bfloat16* act, int M, int N, int K,
                       cudaStream_t s) {
  if (use_pair() && fuse_swiglu() && M >= 256 && N >= 256 && N % 32 == 0) {
    GemmOut out{pre, N};
    out.aux = act;
    out.ldaux = N;
    out.bias = bias;
    return gemm_bf16_pair(GemmOperand{A, lda, false}, GemmOperand{W, ldw, false}, out, M, N, K, 1.0f, EPI_GELU, s);
  }
  const int rc = gemm_fwd_bias(A, lda, W, ldw, pre, N, bias, M, N, K, s);
  return rc ? rc : launch_gelu_fwd(pre, act, static_cast<long long>(M) * N, s);
}

int gemm_dx_dgelu(const __nv_bfloat16* dY, long long ldy, const __nv_bfloat16* W, long long ldw,
                  const __nv_bfloat16* pre, __nv_bfloat16* d_act, __nv_bfloat16* dpre, float* db, int M, int N, int K,
                  cudaStream_t s) {
  if (use_pair() && fuse_swiglu() && M >= 256 && N >= 256 && N % 32 == 0) {
    GemmOut out{dpre, N};
    out.residual = pre;
    out.ldr = N;
    out.colsum = db;
    return gemm_bf16_pair(GemmOperand{dY, ldy, false}, GemmOperand{W, ldw, true}, out, M, N, K, 1.0f, EPI_DGELU,
                          s);
  }
  int rc = gemm_dx(dY, ldy, W, ldw, d_act, N, M, N, K, EPI_STORE_BF16, s);
  if (!rc) rc = launch_gelu_bwd(pre, d_act, dpre, static_cast<long long>(M) * N, s);
  if (!rc && db) rc = launch_bias_grad(dpre, N, db, M, N, s);
  return rc;
}

}  // namespace ops

using namespace ops;

ParamSlice Stage::add_matrix(int rows, int cols, bool freezable) {
  ParamSlice p;
  p.offset = n_params_;
  p.count = static_cast<long long>(rows) * cols;
  p.rows = rows;
  p.cols = cols;
  n_params_ = round_up(n_params_ + p.count, kAlign);
  if (freezable) {
    UnitMatrix m{};
    m.elem_offset = p.offset;
    m.rows = rows;
    m.cols = cols;
    m.unit_offset = total_units_;
    m.tiles_n = (cols + 127) / 128;
    m.units = ((rows + 127) / 128) * m.tiles_n;
    m.pair_offset = pair_capacity_;
    pair_capacity_ += pair_list_capacity((rows + 127) / 128, m.tiles_n);  // even: lists stay int2-aligned
    total_units_ += m.units;
    p.unit_matrix = static_cast<int>(mats_.size());
    mats_.push_back(m);
  }
  return p;
}

ParamSlice Stage::add_dense(long long n) {
  ParamSlice p;
  p.offset = n_params_;
  p.count = n;
  p.rows = 1;
  p.cols = static_cast<int>(n);
  n_params_ = round_up(n_params_ + n, kAlign);
  return p;
}

Stage::Stage(const ModelConfig& cfg, const StageSpec& spec, int device, bool split_backward)
    : cfg_(cfg), spec_(spec), device_(device), split_(split_backward) {
  cudaSetDevice(device);
}

void* Stage::alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaMalloc(&p, std::max<size_t>(bytes, 256)) != cudaSuccess)
    throw std::runtime_error("stage: cudaMalloc of " + std::to_string(bytes) + " bytes failed");
  allocations_.push_back(p);
  return p;
}

void Stage::allocate_parameters(uint64_t seed) {
  master_ = alloc_f32(n_params_);
  weights_ = alloc_bf16(n_params_);
  grad_ = alloc_f32(n_params_);
  stamps_ = static_cast<int*>(alloc(static_cast<size_t>(total_units_) * 4));
  cudaMemset(stamps_, 0, static_cast<size_t>(total_units_) * 4);
  if (const char* e = std::getenv("PF_DW_KERNEL")) {
    const std::string k(e);
    dw_kernel_ = k == "units" ? DW_UNITS : k == "pairs" ? DW_CTA_PAIRS : DW_ROWPAIRS;
  }
  unit_lists_ = static_cast<int*>(
      alloc(static_cast<size_t>((dw_kernel_ == DW_UNITS ? total_units_ : pair_capacity_) + 64) * 4));
  unit_counts_ = static_cast<int*>(alloc(static_cast<size_t>(mats_.size() + 1) * 4));
  mats_dev_ = static_cast<UnitMatrix*>(alloc(mats_.size() * sizeof(UnitMatrix)));
  cudaMemcpy(mats_dev_, mats_.data(), mats_.size() * sizeof(UnitMatrix), cudaMemcpyHostToDevice);
  // matrices N(0, init_std) (fixed seed per stage); families initialise their dense params
  launch_init_normal(master_, weights_, n_unit_params_, cfg_.init_std,
                     seed * 1000003ULL + static_cast<uint64_t>(spec_.stage), nullptr);
  cudaMemset(grad_, 0, static_cast<size_t>(n_params_) * 4);
}

int Stage::build_unit_lists(const uint64_t* frozen_words, cudaStream_t s) {
  const int n = static_cast<int>(mats_.size());
  switch (dw_kernel_) {
    case DW_ROWPAIRS: return launch_mask_to_rowpair_lists(frozen_words, mats_dev_, n, unit_lists_, unit_counts_, s);
    case DW_CTA_PAIRS: return launch_mask_to_pair_lists(frozen_words, mats_dev_, n, unit_lists_, unit_counts_, s);
    default: return launch_mask_to_unit_lists(frozen_words, mats_dev_, n, unit_lists_, unit_counts_, s);
  }
}

LlamaStage::LlamaStage(const ModelConfig& cfg, const StageSpec& spec, int slots, uint64_t seed, int device,
                       bool split_backward)
    : Stage(cfg, spec, device, split_backward) {
  if (cfg.hidden % 128 || cfg.ffn % 128 || cfg.head_dim % 8 || cfg.vocab % 8 || cfg.tokens() % 128)
    throw std::invalid_argument("stage: unsupported model shape (hidden % 128, ffn % 128, vocab % 8, T % 128)");
  const int h = cfg.hidden;
  const int nl = spec.layer_end - spec.layer_begin;
  layers_.resize(static_cast<std::size_t>(nl));
  // freezable 128x128-unit matrices first (contiguous APF state), then dense params
  for (auto& L : layers_) {
    L.wqkv = add_matrix(cfg.qkv_dim(), h, true);
    L.wo = add_matrix(h, cfg.attn_dim(), true);
    L.wgu = add_matrix(2 * cfg.ffn, h, true);
    L.wd = add_matrix(h, cfg.ffn, true);
  }
  if (spec.last) wlm_ = add_matrix(cfg.vocab, h, true);
  end_unit_matrices();
  for (auto& L : layers_) {
    L.g1 = add_dense(h);
    L.g2 = add_dense(h);
  }
  if (spec.last) gf_ = add_dense(h);
  if (spec.first) emb_ = add_matrix(cfg.vocab, h, false);
  allocate_parameters(seed);
  rope_ = static_cast<float2*>(alloc(static_cast<size_t>(cfg.seq) * (cfg.head_dim / 2) * sizeof(float2)));
  launch_rope_table(rope_, cfg.seq, cfg.head_dim, cfg.rope_theta, nullptr);
  // ones for norm gains, N(0, init_std) for the embedding
  for (auto& L : layers_) {
    launch_fill(master_ + L.g1.offset, weights_ + L.g1.offset, h, 1.0f, nullptr);
    launch_fill(master_ + L.g2.offset, weights_ + L.g2.offset, h, 1.0f, nullptr);
  }
  if (spec.last) launch_fill(master_ + gf_.offset, weights_ + gf_.offset, h, 1.0f, nullptr);
  if (spec.first)
    launch_init_normal(master_ + emb_.offset, weights_ + emb_.offset, emb_.count, cfg.init_std,
                       seed * 7919ULL + 17ULL, nullptr);

  const long long T = cfg.tokens();
  auto abf = [&](long long elems) { return alloc_bf16(elems); };
  auto af32 = [&](long long elems) { return alloc_f32(elems); };
  slots_.resize(static_cast<std::size_t>(slots));
  for (auto& sl : slots_) {
    sl.layers.resize(static_cast<std::size_t>(nl));
    for (auto& L : sl.layers) {
      L.x = abf(T * h);
      L.h1 = abf(T * h);
      L.qkv = abf(T * cfg.qkv_dim());
      L.x2 = abf(T * h);
      L.h2 = abf(T * h);
      L.gu = abf(T * 2 * cfg.ffn);
      L.a = abf(T * cfg.ffn);
      L.rstd1 = af32(T);
      L.rstd2 = af32(T);
      L.ao = abf(T * cfg.attn_dim());
      L.lse = af32(static_cast<long long>(cfg.micro_batch) * cfg.n_heads * cfg.seq);
      L.dy = abf(T * h);
      L.dx2 = abf(T * h);
    }
    sl.x_out = abf(T * h);
    if (spec.last) {
      sl.hf = abf(T * h);
      sl.rstdf = af32(T);
      sl.logits = abf(T * cfg.vocab);
    }
  }
  d_a_ = abf(T * cfg.ffn);
  d_h_ = abf(T * h);
  d_attn_ = abf(T * cfg.attn_dim());
  attn_D_ = af32(static_cast<long long>(cfg.micro_batch) * cfg.n_heads * cfg.seq);
  dq_acc_ = af32(T * cfg.attn_dim());
  d_y_ = abf(T * h);
  d_tmp_ = abf(T * h);
  if (cudaDeviceSynchronize() != cudaSuccess) throw std::runtime_error("stage: initialisation kernels failed");
}

LlamaStage::~LlamaStage() { cudaSetDevice(device_); }

Stage::~Stage() {
  cudaSetDevice(device_);
  for (void* p : allocations_) cudaFree(p);
}

long long Stage::matmul_flops_fwd() const {
  long long p = 0;
  for (const auto& m : mats_) p += static_cast<long long>(m.rows) * m.cols;
  return 2LL * cfg_.tokens() * p;
}

int Stage::zero_dense_grads(cudaStream_t s) {
  PF_CUDA(cudaMemsetAsync(grad_ + dense_begin_, 0, static_cast<size_t>(n_params_ - dense_begin_) * 4, s));
  return PF_OK;
}

int LlamaStage::forward(int slot, int microbatch, const int* tokens, const int* targets, const __nv_bfloat16* x_in,
                   float* loss_sum, cudaStream_t s) {
  if (slot < 0 || slot >= static_cast<int>(slots_.size())) return PF_ERR_INVALID;
  Slot& sl = slots_[static_cast<std::size_t>(slot)];
  sl.microbatch = microbatch;
  const int T = cfg_.tokens(), h = cfg_.hidden;
  const size_t act = static_cast<size_t>(T) * h * 2;
  const int nl = static_cast<int>(layers_.size());
  __nv_bfloat16* x0 = nl > 0 ? sl.layers[0].x : sl.x_out;
  if (spec_.first) {
    if (!tokens) return PF_ERR_INVALID;
    PF_TRY(launch_embedding_fwd(tokens, weights_ + emb_.offset, x0, T, h, s));
  } else {
    if (!x_in) return PF_ERR_INVALID;
    PF_CUDA(cudaMemcpyAsync(x0, x_in, act, cudaMemcpyDeviceToDevice, s));
  }
  const float scale = 1.0f / std::sqrt(static_cast<float>(cfg_.head_dim));
  for (int li = 0; li < nl; ++li) {
    SavedLayer& L = sl.layers[static_cast<std::size_t>(li)];
    const LayerParams& P = layers_[static_cast<std::size_t>(li)];
    PF_TRY(launch_rmsnorm_fwd(L.x, weights_ + P.g1.offset, L.h1, L.rstd1, T, h, cfg_.norm_eps, s));
    PF_TRY(gemm_fwd_rope(L.h1, h, weights_ + P.wqkv.offset, h, L.qkv, rope_, T, cfg_.seq, cfg_.n_heads,
                         cfg_.n_kv_heads, cfg_.head_dim, h, s));
    PF_TRY(launch_flash_attn_fwd(L.qkv, L.ao, cfg_.attn_dim(), L.lse, cfg_.micro_batch, cfg_.seq, cfg_.n_heads,
                                 cfg_.n_kv_heads, cfg_.head_dim, scale, true, s));
    L.attn_out = L.ao;
    L.attn_ld = cfg_.attn_dim();
    PF_TRY(gemm_fwd_resid(L.attn_out, L.attn_ld, weights_ + P.wo.offset, cfg_.attn_dim(), L.x2, L.x, h, T, h,
                          cfg_.attn_dim(), s));
    PF_TRY(launch_rmsnorm_fwd(L.x2, weights_ + P.g2.offset, L.h2, L.rstd2, T, h, cfg_.norm_eps, s));
    // bench.py roofline probe: brackets the gate|up GEMM launch alone (with its fused SwiGLU
    // epilogue when that path is taken, else without the separate activation kernel)
    const bool probe = probe_kind() == PROBE_GATE_UP_GEMM;
    if (probe && !(use_pair() && fuse_swiglu_fwd(h))) {
      probe_begin(s);
      PF_TRY(gemm_fwd(L.h2, h, weights_ + P.wgu.offset, h, L.gu, 2 * cfg_.ffn, T, 2 * cfg_.ffn, h, EPI_STORE_BF16, s));
      probe_end(s);
      PF_TRY(launch_swiglu_fwd(L.gu, L.a, T, cfg_.ffn, s));
    } else {
      if (probe) probe_begin(s);
      PF_TRY(gemm_fwd_swiglu(L.h2, h, weights_ + P.wgu.offset, h, L.gu, L.a, T, cfg_.ffn, h, s));
      if (probe) probe_end(s);
    }
    __nv_bfloat16* next = li + 1 < nl ? sl.layers[static_cast<std::size_t>(li + 1)].x : sl.x_out;
    PF_TRY(gemm_fwd_resid(L.a, cfg_.ffn, weights_ + P.wd.offset, cfg_.ffn, next, L.x2, h, T, h, cfg_.ffn, s));
  }
  if (spec_.last) {
    if (!targets || !loss_sum) return PF_ERR_INVALID;
    PF_TRY(launch_rmsnorm_fwd(sl.x_out, weights_ + gf_.offset, sl.hf, sl.rstdf, T, h, cfg_.norm_eps, s));
    PF_TRY(gemm_fwd(sl.hf, h, weights_ + wlm_.offset, h, sl.logits, cfg_.vocab, T, cfg_.vocab, h, EPI_STORE_BF16, s));
    // mean token loss of the microbatch; dlogits = (softmax - onehot) / T in place
    PF_TRY(launch_cross_entropy(sl.logits, targets, loss_sum, T, cfg_.vocab, 1.0f / T, 1.0f / T, s));
  }
  return PF_OK;
}

DwGemm Stage::dw_item(const ParamSlice& w, const __nv_bfloat16* dy, long long ldy, const __nv_bfloat16* x,
                      long long ldx, int K) const {
  const UnitMatrix& m = mats_[static_cast<std::size_t>(w.unit_matrix)];
  // dW[out, in] (+)= dY^T . X over the unfrozen units; both operands MN-major (no transposes)
  return DwGemm{dy, ldy, x, ldx, grad_ + w.offset, w.cols, w.rows, w.cols, K,
                unit_lists_ + (dw_kernel_ == DW_UNITS ? m.unit_offset : m.pair_offset), unit_counts_ + w.unit_matrix,
                m.unit_offset};
}

int LlamaStage::backward(int slot, const int* tokens, const uint64_t* frozen_words, const __nv_bfloat16* dy,
                    __nv_bfloat16* dx_out, int stamp, cudaStream_t s) {
  if (slot < 0 || slot >= static_cast<int>(slots_.size()) || (!frozen_words && !split_)) return PF_ERR_INVALID;
  Slot& sl = slots_[static_cast<std::size_t>(slot)];
  const int T = cfg_.tokens(), h = cfg_.hidden, ffn = cfg_.ffn;
  const int nl = static_cast<int>(layers_.size());
  // K5p: this microbatch's unit mask -> per-matrix pair lists of unfrozen units (W does it when split)
  if (!split_)
    PF_TRY(build_unit_lists(frozen_words, s));
  // every layer's output gradient lands in its slot buffer; the top layer's is the incoming
  // gradient itself when W runs inside this action (split: copied, the buffer is reused)
  __nv_bfloat16* top = nl > 0 ? sl.layers[static_cast<std::size_t>(nl - 1)].dy : d_y_;
  const __nv_bfloat16* dcur = dy;
  if (spec_.last) {
    PF_TRY(gemm_dx(sl.logits, cfg_.vocab, weights_ + wlm_.offset, h, d_h_, h, T, h, cfg_.vocab, EPI_STORE_BF16, s));
    PF_TRY(launch_rmsnorm_bwd(sl.x_out, weights_ + gf_.offset, sl.rstdf, d_h_, nullptr, top, grad_ + gf_.offset, T,
                              h, s));
    dcur = top;
  } else if (split_ && nl > 0 && dcur) {
    PF_CUDA(cudaMemcpyAsync(top, dcur, static_cast<size_t>(T) * h * 2, cudaMemcpyDeviceToDevice, s));
    dcur = top;
  }
  if (!dcur) return PF_ERR_INVALID;
  for (int li = nl - 1; li >= 0; --li) {
    SavedLayer& L = sl.layers[static_cast<std::size_t>(li)];
    const LayerParams& P = layers_[static_cast<std::size_t>(li)];
    L.dy_w = dcur;
    // d(gate|up) over gu and dqkv over qkv (both dead after their use here), dx2 kept for W
    __nv_bfloat16* dgu = L.gu;
    __nv_bfloat16* dx2 = L.dx2;
    __nv_bfloat16* dqkv = L.qkv;
    // MLP
    PF_TRY(gemm_dx_dswiglu(dcur, h, weights_ + P.wd.offset, ffn, L.gu, d_a_, dgu, T, ffn, h, s));
    PF_TRY(gemm_dx(dgu, 2 * ffn, weights_ + P.wgu.offset, h, d_h_, h, T, h, 2 * ffn, EPI_STORE_BF16, s));
    PF_TRY(launch_rmsnorm_bwd(L.x2, weights_ + P.g2.offset, L.rstd2, d_h_, dcur, dx2, grad_ + P.g2.offset, T, h, s));
    // attention
    PF_TRY(gemm_dx(dx2, h, weights_ + P.wo.offset, cfg_.attn_dim(), d_attn_, cfg_.attn_dim(), T, cfg_.attn_dim(), h,
                   EPI_STORE_BF16, s));
    // dq|dk|dv with the RoPE backward, packed over qkv (the key block's owner writes dk / dv in
    // place once it no longer reads k / v; dq follows from the fp32 accumulator)
    PF_TRY(launch_flash_attn_bwd(L.qkv, L.ao, d_attn_, L.lse, attn_D_, dq_acc_, dqkv, rope_, cfg_.micro_batch,
                                 cfg_.seq, cfg_.n_heads, cfg_.n_kv_heads, cfg_.head_dim,
                                 1.0f / std::sqrt(static_cast<float>(cfg_.head_dim)), true, s));
    PF_TRY(gemm_dx(dqkv, cfg_.qkv_dim(), weights_ + P.wqkv.offset, h, d_h_, h, T, h, cfg_.qkv_dim(),
                   EPI_STORE_BF16, s));
    __nv_bfloat16* out;
    if (li > 0) out = sl.layers[static_cast<std::size_t>(li - 1)].dy;
    else out = spec_.first ? d_tmp_ : dx_out;
    if (!out) return PF_ERR_INVALID;
    PF_TRY(launch_rmsnorm_bwd(L.x, weights_ + P.g1.offset, L.rstd1, d_h_, dx2, out, grad_ + P.g1.offset, T, h, s));
    dcur = out;
  }
  if (spec_.first) PF_TRY(launch_embedding_bwd(tokens, dcur, grad_ + emb_.offset, T, h, s));
  else if (nl == 0 && dx_out && dcur != dx_out)
    PF_CUDA(cudaMemcpyAsync(dx_out, dcur, static_cast<size_t>(T) * h * 2, cudaMemcpyDeviceToDevice, s));
  // K3: all masked weight gradients of the microbatch in one launch (split: in W)
  if (!split_) PF_TRY(weight_grads(sl, stamp, s));
  return PF_OK;
}

int LlamaStage::weight_grads(Slot& sl, int stamp, cudaStream_t s) {
  const int T = cfg_.tokens(), h = cfg_.hidden, ffn = cfg_.ffn;
  std::vector<DwGemm> items;
  items.reserve(4 * layers_.size() + 1);
  if (spec_.last) items.push_back(dw_item(wlm_, sl.logits, cfg_.vocab, sl.hf, h, T));
  for (int li = static_cast<int>(layers_.size()) - 1; li >= 0; --li) {
    const SavedLayer& L = sl.layers[static_cast<std::size_t>(li)];
    const LayerParams& P = layers_[static_cast<std::size_t>(li)];
    items.push_back(dw_item(P.wd, L.dy_w, h, L.a, ffn, T));
    items.push_back(dw_item(P.wgu, L.gu, 2LL * ffn, L.h2, h, T));
    items.push_back(dw_item(P.wo, L.dx2, h, L.attn_out, L.attn_ld, T));
    items.push_back(dw_item(P.wqkv, L.qkv, cfg_.qkv_dim(), L.h1, h, T));
  }
  return run_dw(items, stamp, s);
}

int LlamaStage::backward_weight(int slot, const uint64_t* frozen_words, int stamp, cudaStream_t s) {
  if (!split_ || slot < 0 || slot >= static_cast<int>(slots_.size()) || !frozen_words) return PF_ERR_INVALID;
  PF_TRY(build_unit_lists(frozen_words, s));
  return weight_grads(slots_[static_cast<std::size_t>(slot)], stamp, s);
}

int Stage::optimizer_step(const OptimCfg& oc, int microbatches, int stamp, bool apf, float apf_alpha,
                          float apf_threshold, cudaStream_t s) {
  if (apf && !apf_ema_) {
    PF_CUDA(cudaMalloc(&apf_ema_, static_cast<size_t>(n_unit_params_) * 4));
    PF_CUDA(cudaMalloc(&apf_ema_abs_, static_cast<size_t>(n_unit_params_) * 4));
    PF_CUDA(cudaMalloc(&apf_eligible_, static_cast<size_t>(total_units_) * 4));
    allocations_.push_back(apf_ema_);
    allocations_.push_back(apf_ema_abs_);
    allocations_.push_back(apf_eligible_);
    PF_CUDA(cudaMemsetAsync(apf_ema_, 0, static_cast<size_t>(n_unit_params_) * 4, s));
    PF_CUDA(cudaMemsetAsync(apf_ema_abs_, 0, static_cast<size_t>(n_unit_params_) * 4, s));
  }
  if (oc.adamw && !adam_m_) {
    PF_CUDA(cudaMalloc(&adam_m_, static_cast<size_t>(n_params_) * 4));
    PF_CUDA(cudaMalloc(&adam_v_, static_cast<size_t>(n_params_) * 4));
    PF_CUDA(cudaMalloc(&unit_steps_, static_cast<size_t>(std::max(1, total_units_)) * 4));
    allocations_.push_back(adam_m_);
    allocations_.push_back(adam_v_);
    allocations_.push_back(unit_steps_);
    PF_CUDA(cudaMemsetAsync(adam_m_, 0, static_cast<size_t>(n_params_) * 4, s));
    PF_CUDA(cudaMemsetAsync(adam_v_, 0, static_cast<size_t>(n_params_) * 4, s));
    PF_CUDA(cudaMemsetAsync(unit_steps_, 0, static_cast<size_t>(std::max(1, total_units_)) * 4, s));
  }
  const float inv_m = 1.0f / static_cast<float>(microbatches);
  OptimArgs a{};
  a.master = master_;
  a.weights = weights_;
  a.grad = grad_;
  a.unit_stamp = stamps_;
  a.stamp = stamp;
  a.scale = oc.adamw ? inv_m : oc.lr * inv_m;
  a.mats = mats_dev_;
  a.nmats = static_cast<int>(mats_.size());
  a.total_units = total_units_;
  a.apf_ema = apf ? apf_ema_ : nullptr;
  a.apf_ema_abs = apf ? apf_ema_abs_ : nullptr;
  a.apf_alpha = apf_alpha;
  a.apf_threshold = apf_threshold;
  a.apf_eligible = apf ? apf_eligible_ : nullptr;
  a.apf_elem_base = 0;
  a.adamw = oc.adamw;
  a.adam_m = adam_m_;
  a.adam_v = adam_v_;
  a.unit_steps = unit_steps_;
  a.lr = oc.lr;
  a.beta1 = static_cast<float>(oc.beta1);
  a.beta2 = static_cast<float>(oc.beta2);
  a.beta1_d = oc.beta1;
  a.beta2_d = oc.beta2;
  a.one_minus_beta1 = static_cast<float>(1.0 - oc.beta1);
  a.one_minus_beta2 = static_cast<float>(1.0 - oc.beta2);
  a.eps = oc.eps;
  a.weight_decay = oc.weight_decay;
  PF_TRY(launch_masked_sgd_units(a, s));
  const long long nd = n_params_ - dense_begin_;
  if (!oc.adamw)
    return launch_sgd_dense(master_ + dense_begin_, weights_ + dense_begin_, grad_ + dense_begin_, nd, a.scale, s);
  ++dense_steps_;
  const double bc1 = 1.0 - std::pow(oc.beta1, dense_steps_);
  const double bc2 = 1.0 - std::pow(oc.beta2, dense_steps_);
  return launch_adamw_dense(master_ + dense_begin_, weights_ + dense_begin_, grad_ + dense_begin_,
                            adam_m_ + dense_begin_, adam_v_ + dense_begin_, nd, inv_m, oc.lr, a.beta1, a.beta2,
                            a.one_minus_beta1, a.one_minus_beta2, oc.eps, oc.weight_decay, bc1, bc2, s);
}

}  // namespace pf

namespace pf {

std::unique_ptr<Stage> make_vit_stage(const ModelConfig& cfg, const StageSpec& spec, int slots, uint64_t seed,
                                      int device, bool split_backward);

std::unique_ptr<Stage> make_stage(const ModelConfig& cfg, const StageSpec& spec, int slots, uint64_t seed,
                                  int device, bool split_backward) {
  set_pdl_default(cfg.family == 1);  // PDL pays on the ViT step's many small kernels only
  if (cfg.family == 1) return make_vit_stage(cfg, spec, slots, seed, device, split_backward);
  if (cfg.family != 0) throw std::invalid_argument("stage: unknown model family");
  return std::make_unique<LlamaStage>(cfg, spec, slots, seed, device, split_backward);
}

}  // namespace pf
