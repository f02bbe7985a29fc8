// ViT encoder glue kernels (vit_kernels.cu). bf16 activations, fp32 statistics and
// parameter gradients (gradients accumulate: +=).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace pf {

// y = LayerNorm(x) * g + b per row of h; saves mean and rstd per row
int launch_layernorm_fwd(const __nv_bfloat16* x, const __nv_bfloat16* g, const __nv_bfloat16* b, __nv_bfloat16* y,
                         float* mean, float* rstd, int T, int h, float eps, cudaStream_t s);
// dx = residual + LayerNorm backward; dg += sum dy * xhat, db += sum dy (either may be nullptr)
// dsum (may be nullptr): += column sums of the bf16 dx (the bias gradient of the linear layer
// whose output gradient dx is), computed in the same pass on the fused path (h = 256, 512, 1024)
int launch_layernorm_bwd(const __nv_bfloat16* x, const __nv_bfloat16* g, const float* mean, const float* rstd,
                         const __nv_bfloat16* dy, const __nv_bfloat16* residual, __nv_bfloat16* dx, float* dg,
                         float* db, float* dsum, int T, int h, cudaStream_t s);
// db[c] += sum_t dy[t, c] (bias gradient of a linear layer)
// Bidirectional attention for S <= 64, head_dim 64 (vit_attention.cu): qkv packed [B S, 3 nh 64],
// out [B S, nh 64], lse fp32 [B][nh][S]; the backward writes dq|dk|dv packed into dqkv (may alias qkv).
int launch_vit_attn_fwd(const __nv_bfloat16* qkv, __nv_bfloat16* out, float* lse, int B, int S, int nh, int hd,
                        float scale, cudaStream_t s);
// dbias (nullable): += column sums of the packed dq|dk|dv (the qkv bias gradient), from the same CTAs
int launch_vit_attn_bwd(const __nv_bfloat16* qkv, const __nv_bfloat16* out, const __nv_bfloat16* dout,
                        const float* lse, __nv_bfloat16* dqkv, float* dbias, int B, int S, int nh, int hd, float scale,
                        cudaStream_t s);

int launch_bias_grad(const __nv_bfloat16* dy, long long ldy, float* db, int T, int n, cudaStream_t s);
// act = GELU(pre) (erf form); dpre = dact * GELU'(pre)
int launch_gelu_fwd(const __nv_bfloat16* pre, __nv_bfloat16* act, long long n, cudaStream_t s);
int launch_gelu_bwd(const __nv_bfloat16* pre, const __nv_bfloat16* dact, __nv_bfloat16* dpre, long long n,
                    cudaStream_t s);
// C[M, N] += bias (for GEMMs whose epilogue has no bias: the 1-CTA fallback)
int launch_add_bias(__nv_bfloat16* c, long long ldc, const __nv_bfloat16* bias, int M, int N, cudaStream_t s);
// x [B*S, h] from patch embeddings E [B*(S-1), h], the patch bias, cls token and positions [S, h]
int launch_vit_embed_fwd(const __nv_bfloat16* E, const __nv_bfloat16* pbias, const __nv_bfloat16* cls,
                         const __nv_bfloat16* pos, __nv_bfloat16* x, int B, int S, int h, cudaStream_t s);
int launch_vit_embed_bwd(const __nv_bfloat16* dx, __nv_bfloat16* dE, float* dpos, float* dcls, float* dpbias, int B,
                         int S, int h, cudaStream_t s);
// cls rows (token 0 of each image) out of / back into a [B*S, h] activation (scatter zero-fills)
int launch_gather_rows(const __nv_bfloat16* x, __nv_bfloat16* out, int B, int S, int h, cudaStream_t s);
int launch_scatter_rows(const __nv_bfloat16* src, __nv_bfloat16* dx, int B, int S, int h, cudaStream_t s);
// deterministic synthetic pixels in [-1, 1) for the patch input [B*(S-1), patch_dim]
int launch_synthetic_patches(__nv_bfloat16* out, long long n, uint64_t seed, cudaStream_t s);

}  // namespace pf
