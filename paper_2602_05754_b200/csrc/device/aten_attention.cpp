// Causal GQA attention for the LLaMA stage (K7 glue), delegated to ATen's
// fused-attention ops (library code, like cuBLAS; the only non-hand-written
// kernels on the step). Backend: cuDNN fused attention (Blackwell kernels) by
// default, FlashAttention-2 with PF_ATTN_BACKEND=flash or if cuDNN rejects the
// shape. q/k/v are zero-copy views into the packed qkv activation
// [T, (nh + 2 nkv) hd]; for cuDNN, K/V are expanded to nh heads (and dK/dV
// group-summed). Outputs stay on the caller's stream.
#include <ATen/ATen.h>
#include <c10/cuda/CUDAGuard.h>
#include <c10/cuda/CUDAStream.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <string>

#include "attention.hpp"
#include "pf_status.h"

namespace pf {

struct AttnState {
  at::Tensor out, lse, cum_q, cum_k, seed, offset;
  at::Tensor dq, dk, dv;
  int64_t max_q = 0, max_k = 0;
  bool cudnn = false;
  bool causal = true;
  int rep = 1;  // K/V head expansion used for this forward (1 = native GQA)
};

namespace {

thread_local std::string g_attn_err;

// 1 = cuDNN, 0 = flash; cuDNN is disabled for the process after its first failure
int g_backend = -1;

int backend() {
  if (g_backend < 0) {
    const char* e = std::getenv("PF_ATTN_BACKEND");
    g_backend = (e && std::string(e) == "flash") ? 0 : 1;
  }
  return g_backend;
}

struct Views {
  at::Tensor q, k, v;
};

Views make_views(const void* qkv, int B, int S, int nh, int nkv, int hd) {
  const auto opts = at::TensorOptions().dtype(at::kBFloat16).device(at::kCUDA, c10::cuda::current_device());
  const int64_t W = static_cast<int64_t>(nh + 2 * nkv) * hd;
  auto* base = static_cast<at::BFloat16*>(const_cast<void*>(qkv));
  auto view = [&](int64_t off, int heads) {
    return at::from_blob(base + off, {B, S, heads, hd}, {S * W, W, hd, 1}, opts).transpose(1, 2);
  };
  return Views{view(0, nh), view(static_cast<int64_t>(nh) * hd, nkv), view(static_cast<int64_t>(nh + nkv) * hd, nkv)};
}

at::Tensor expand_heads(const at::Tensor& t, int rep) { return rep == 1 ? t : t.repeat_interleave(rep, 1); }

c10::cuda::CUDAStream wrap(cudaStream_t s) {
  return c10::cuda::getStreamFromExternal(s, c10::cuda::current_device());
}

}  // namespace

AttnState* attn_state_new() { return new AttnState(); }
void attn_state_free(AttnState* st) { delete st; }
const char* attn_last_error() { return g_attn_err.c_str(); }
int attn_backend_is_cudnn() { return backend(); }

int attn_fwd(AttnState* st, const void* qkv, int B, int S, int nh, int nkv, int hd, float scale, void** out,
             long long* out_token_stride, cudaStream_t stream, bool causal) {
  try {
    c10::cuda::CUDAStreamGuard guard(wrap(stream));
    const auto v = make_views(qkv, B, S, nh, nkv, hd);
    at::Tensor o;
    st->cudnn = false;
    st->causal = causal;
    if (backend() == 1) {
      try {
        // native GQA (nkv < nh K/V heads) when cuDNN accepts it, else expanded K/V
        static int native_gqa = -1;
        const int full_rep = nh / nkv;
        auto run = [&](int rep) {
          return at::_scaled_dot_product_cudnn_attention(v.q, expand_heads(v.k, rep), expand_heads(v.v, rep),
                                                         std::nullopt, true, 0.0, causal, false,
                                                         static_cast<double>(scale));
        };
        decltype(run(1)) r;
        if (full_rep > 1 && native_gqa != 0) {
          try {
            r = run(1);
            native_gqa = 1;
          } catch (const std::exception&) {
            native_gqa = 0;
          }
        }
        st->rep = (full_rep > 1 && native_gqa == 1) ? 1 : full_rep;
        if (full_rep == 1 || native_gqa == 0) r = run(st->rep);
        o = std::get<0>(r);
        st->lse = std::get<1>(r);
        st->cum_q = std::get<2>(r);
        st->cum_k = std::get<3>(r);
        st->max_q = std::get<4>(r).expect_int();
        st->max_k = std::get<5>(r).expect_int();
        st->seed = std::get<6>(r);
        st->offset = std::get<7>(r);
        st->cudnn = true;
      } catch (const std::exception& e) {
        g_backend = 0;  // fall back to the flash kernels for the rest of the run
        g_attn_err = std::string("cudnn attention unavailable, using flash: ") + e.what();
      }
    }
    if (!st->cudnn) {
      auto r = at::_scaled_dot_product_flash_attention(v.q, v.k, v.v, 0.0, causal, false, static_cast<double>(scale));
      o = std::get<0>(r);
      st->lse = std::get<1>(r);
      st->cum_q = std::get<2>(r);
      st->cum_k = std::get<3>(r);
      st->max_q = std::get<4>(r).expect_int();
      st->max_k = std::get<5>(r).expect_int();
      st->seed = std::get<6>(r);
      st->offset = std::get<7>(r);
    }
    // Wo GEMM wants [T, nh*hd] row-major = [B, S, H, D] contiguous
    at::Tensor bshd = o.transpose(1, 2);
    if (!bshd.is_contiguous()) o = bshd.contiguous().transpose(1, 2);
    st->out = o;
    *out = st->out.data_ptr();
    *out_token_stride = st->out.stride(2);
    return PF_OK;
  } catch (const std::exception& e) {
    g_attn_err = e.what();
    return PF_ERR_CUDA;
  }
}

int attn_bwd(AttnState* st, const void* qkv, const void* dout, int B, int S, int nh, int nkv, int hd, float scale,
             AttnGrads* g, cudaStream_t stream) {
  try {
    c10::cuda::CUDAStreamGuard guard(wrap(stream));
    const auto v = make_views(qkv, B, S, nh, nkv, hd);
    const auto opts = at::TensorOptions().dtype(at::kBFloat16).device(at::kCUDA, c10::cuda::current_device());
    auto* dptr = static_cast<at::BFloat16*>(const_cast<void*>(dout));
    const int64_t W = static_cast<int64_t>(nh) * hd;
    at::Tensor go = at::from_blob(dptr, {B, S, nh, hd}, {S * W, W, hd, 1}, opts).transpose(1, 2);
    at::Tensor dq, dk, dv;
    int rep = 1;
    if (st->cudnn) {
      rep = st->rep;
      auto r = at::_scaled_dot_product_cudnn_attention_backward(
          go, v.q, expand_heads(v.k, rep), expand_heads(v.v, rep), st->out, st->lse, st->seed, st->offset,
          at::Tensor(), st->cum_q, st->cum_k, st->max_q, st->max_k, 0.0, st->causal, static_cast<double>(scale));
      dq = std::get<0>(r);
      dk = std::get<1>(r);  // nkv * rep heads; the pack kernel sums each group of rep
      dv = std::get<2>(r);
    } else {
      auto r = at::_scaled_dot_product_flash_attention_backward(go, v.q, v.k, v.v, st->out, st->lse, st->cum_q,
                                                                st->cum_k, st->max_q, st->max_k, 0.0, st->causal, st->seed,
                                                                st->offset, static_cast<double>(scale));
      dq = std::get<0>(r);
      dk = std::get<1>(r);
      dv = std::get<2>(r);
    }
    // strided [B, H, S, D] views straight into the pack kernel (no copies)
    st->dq = dq;
    st->dk = dk;
    st->dv = dv;
    g->dq = dq.data_ptr();
    g->dk = dk.data_ptr();
    g->dv = dv.data_ptr();
    g->q_b = dq.stride(0);
    g->q_h = dq.stride(1);
    g->q_t = dq.stride(2);
    g->k_b = dk.stride(0);
    g->k_h = dk.stride(1);
    g->k_t = dk.stride(2);
    g->v_b = dv.stride(0);
    g->v_h = dv.stride(1);
    g->v_t = dv.stride(2);
    g->rep = rep;
    return PF_OK;
  } catch (const std::exception& e) {
    g_attn_err = e.what();
    return PF_ERR_CUDA;
  }
}

void attn_release_keep_out(AttnState* st) {
  st->lse = at::Tensor();
  st->dq = at::Tensor();
  st->dk = at::Tensor();
  st->dv = at::Tensor();
}

void attn_release(AttnState* st) {
  st->out = at::Tensor();
  st->lse = at::Tensor();
  st->dq = at::Tensor();
  st->dk = at::Tensor();
  st->dv = at::Tensor();
}

}  // namespace pf
