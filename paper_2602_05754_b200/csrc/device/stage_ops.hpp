// GEMM call patterns shared by the stage families (defined in stage.cpp): the
// CTA-pair kernel for the large K1 / K2 GEMMs, the 1-CTA kernel below its tile size.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "pf_device_internal.hpp"

namespace pf {
namespace ops {

bool use_pair();
// SwiGLU / GELU fused in the CTA-pair GEMM epilogues (PF_FUSE_SWIGLU=0 turns both off)
bool fuse_swiglu();
// Y[M,N] (op)= A[M,K] . W[N,K]^T, both K-major
int gemm_fwd(const __nv_bfloat16* A, long long lda, const __nv_bfloat16* W, long long ldw, void* C, long long ldc,
             int M, int N, int K, int epi, cudaStream_t s);
// Y = R + A . W^T (residual fused in the CTA-pair epilogue)
int gemm_fwd_resid(const __nv_bfloat16* A, long long lda, const __nv_bfloat16* W, long long ldw, __nv_bfloat16* C,
                   const __nv_bfloat16* R, long long ld, int M, int N, int K, cudaStream_t s);
// Y = A . W^T + bias, and Y = R + A . W^T + bias (bias fused in the CTA-pair epilogue)
int gemm_fwd_bias(const __nv_bfloat16* A, long long lda, const __nv_bfloat16* W, long long ldw, __nv_bfloat16* C,
                  long long ldc, const __nv_bfloat16* bias, int M, int N, int K, cudaStream_t s);
int gemm_fwd_resid_bias(const __nv_bfloat16* A, long long lda, const __nv_bfloat16* W, long long ldw,
                        __nv_bfloat16* C, const __nv_bfloat16* R, long long ld, const __nv_bfloat16* bias, int M,
                        int N, int K, cudaStream_t s);
// qkv = A . Wqkv^T with rotate-half RoPE on the q and k heads (fused in the CTA-pair epilogue when
// head_dim == 64, else GEMM + rope_fwd_kernel)
int gemm_fwd_rope(const __nv_bfloat16* A, long long lda, const __nv_bfloat16* W, long long ldw, __nv_bfloat16* qkv,
                  const float2* rope, int M, int seq, int nh, int nkv, int hd, int K, cudaStream_t s);
// ViT MLP: pre = A . W1^T + bias and act = gelu(pre) (GELU fused in the CTA-pair epilogue);
// dpre = (dY . W2) * gelu'(pre), dpre may alias pre (d_act scratch only on the unfused path)
int gemm_fwd_bias_gelu(const __nv_bfloat16* A, long long lda, const __nv_bfloat16* W, long long ldw,
                       const __nv_bfloat16* bias, __nv_bfloat16* pre, __nv_bfloat16* act, int M, int N, int K,
                       cudaStream_t s);
// db (may be nullptr) += column sums of dpre (the fc1 bias gradient), in the epilogue when fused
int gemm_dx_dgelu(const __nv_bfloat16* dY, long long ldy, const __nv_bfloat16* W, long long ldw,
                  const __nv_bfloat16* pre, __nv_bfloat16* d_act, __nv_bfloat16* dpre, float* db, int M, int N, int K,
                  cudaStream_t s);
// dX[M=T, N=in] = dY[T, K=out] . W[out, in]   (W read MN-major, no transpose)
int gemm_dx(const __nv_bfloat16* dY, long long ldy, const __nv_bfloat16* W, long long ldw, void* C, long long ldc,
            int M, int N, int K, int epi, cudaStream_t s);

}  // namespace ops
}  // namespace pf
