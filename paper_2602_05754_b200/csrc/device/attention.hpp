// Opaque bridge to the ATen flash-attention glue (aten_attention.cpp), so the
// CUDA translation units never include torch headers.
#pragma once
#include <cuda_runtime.h>

namespace pf {

struct AttnState;

// Gradients w.r.t. q, k, v as [B, H, S, D] views with element strides; dk/dv
// carry nkv * rep heads when K/V were expanded for the library call.
struct AttnGrads {
  const void* dq;
  const void* dk;
  const void* dv;
  long long q_b, q_t, q_h, k_b, k_t, k_h, v_b, v_t, v_h;
  int rep;
};

AttnState* attn_state_new();
void attn_state_free(AttnState* st);
const char* attn_last_error();

// qkv: packed [B*S, (nh + 2 nkv) hd] bf16 after RoPE. *out receives the
// attention output [B*S, nh*hd] (row stride *out_token_stride), owned by st.
// causal = false: bidirectional (ViT encoder); the backward uses the forward's mode.
int attn_fwd(AttnState* st, const void* qkv, int B, int S, int nh, int nkv, int hd, float scale, void** out,
             long long* out_token_stride, cudaStream_t stream, bool causal = true);
// dout: [B*S, nh*hd] gradient of the attention output. Gradients stay owned by st.
int attn_bwd(AttnState* st, const void* qkv, const void* dout, int B, int S, int nh, int nkv, int hd, float scale,
             AttnGrads* g, cudaStream_t stream);
// release saved forward tensors (after the backward consumed them)
void attn_release(AttnState* st);
// Split backward: drop the softmax statistics and dQ/dK/dV after B but keep the
// attention output, which W still reads as the X operand of dWo.
void attn_release_keep_out(AttnState* st);
// 1 while the cuDNN fused-attention backend is in use, 0 for flash-attention
int attn_backend_is_cudnn();

}  // namespace pf
