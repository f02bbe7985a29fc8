// Bidirectional attention for short sequences (ViT-L/32: S = 50 tokens, head_dim 64),
// forward and backward, one CTA per (image, head).
//
// At S <= 64 a head's Q, K, V (and O, dO) are 8 KB tiles: the whole problem of one
// (image, head) fits in shared memory, S = QK^T is one 64 x 64 tile and no online
// softmax is needed. The op is HBM-bound (forward: read Q, K, V, write O, 4 x 6.5 MB per
// layer and microbatch; backward: read Q, K, V, dO, write dQ, dK, dV), so the 64 x 64 x 64
// products run on warp-level MMAs (mma.sync m16n8k16, bf16 in, fp32 accumulate) straight
// from shared memory; a 128-row tcgen05 tile would be half padding here. The generic fused
// attention (cuDNN) spent 18.5 us forward and 62 us backward per layer on this shape.
//
// Layout: qkv packed [T = B S, 3 nh hd] (q heads, then k, then v), O [T, nh hd], LSE fp32
// [B][nh][S] (natural log of the row sums, in scaled-score units). The backward writes dQ,
// dK, dV into a packed dqkv (may alias qkv: each CTA reads its head's tiles before writing).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernel_util.cuh"
#include "ptx.cuh"
#include "vit_kernels.cuh"

namespace pf {

namespace {

constexpr int kS = 64;      // padded sequence
constexpr int kD = 64;      // head dim
constexpr int kLd = kD + 8;  // smem row stride (bf16): 144 B rows, conflict-free ldmatrix
constexpr int kThreads = 128;

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void ldsm_x4(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(smem_addr(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(smem_addr(p)));
}
// D (16x8 fp32) += A (16x16 bf16, row) * B (16x8 bf16, col)
__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// A fragment (16 x 16) of a row-major [rows][kLd] tile at (r0, k0)
__device__ __forceinline__ void load_a(uint32_t (&a)[4], const __nv_bfloat16* t, int r0, int k0, int lane) {
  const int m = lane >> 3;
  ldsm_x4(a[0], a[1], a[2], a[3], t + (r0 + (lane & 7) + (m & 1) * 8) * kLd + k0 + (m >> 1) * 8);
}
// A fragment (16 rows r0.. x 16 k0..) of the TRANSPOSE of a row-major [k][r] tile
__device__ __forceinline__ void load_a_t(uint32_t (&a)[4], const __nv_bfloat16* t, int r0, int k0, int lane) {
  const int m = lane >> 3;  // a0: (r, k) = (0..7, 0..7), a1: (8.., 0..), a2: (0.., 8..), a3: (8.., 8..)
  ldsm_x4_t(a[0], a[1], a[2], a[3], t + (k0 + (lane & 7) + (m >> 1) * 8) * kLd + r0 + (m & 1) * 8);
}
// B fragments (16 k0.. x 8 n) for two n tiles n0, n0 + 8, when B^T is stored row-major [n][k]
__device__ __forceinline__ void load_b_nk(uint32_t (&b)[4], const __nv_bfloat16* t, int n0, int k0, int lane) {
  const int m = lane >> 3;  // b[0], b[1]: n tile n0 (k 0..7, 8..15); b[2], b[3]: n tile n0 + 8
  ldsm_x4(b[0], b[1], b[2], b[3], t + (n0 + (lane & 7) + (m >> 1) * 8) * kLd + k0 + (m & 1) * 8);
}
// B fragments (16 k0.. x 8 n) for two n tiles n0, n0 + 8, when B is stored row-major [k][n]
__device__ __forceinline__ void load_b_kn(uint32_t (&b)[4], const __nv_bfloat16* t, int n0, int k0, int lane) {
  const int m = lane >> 3;
  ldsm_x4_t(b[0], b[1], b[2], b[3], t + (k0 + (lane & 7) + (m & 1) * 8) * kLd + n0 + (m >> 1) * 8);
}

__device__ __forceinline__ uint32_t pack2(float lo, float hi) { return pack_bf16x2(lo, hi); }

// rows [0, S) of a head's 64 columns at `col` of a [*, ld] bf16 matrix -> smem tile (zero-padded),
// by cp.async: every tile load of a CTA is in flight at once (cp_async_wait_all before use)
__device__ __forceinline__ void load_tile(__nv_bfloat16* t, const __nv_bfloat16* g, long long row0, long long ld,
                                          int col, int S) {
#pragma unroll
  for (int i = threadIdx.x; i < kS * (kD / 8); i += kThreads) {
    const int r = i >> 3, c = (i & 7) * 8;
    const bool ok = r < S;
    const __nv_bfloat16* src = g + (row0 + (ok ? r : 0)) * ld + col + c;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(t + r * kLd + c)), "l"(src),
                 "r"(ok ? 16 : 0)
                 : "memory");
  }
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// S = scale * Q K^T for the warp's 16 query rows (8 key tiles of 8), keys >= S masked to -inf
__device__ __forceinline__ void scores(float (&s)[8][4], const __nv_bfloat16* Qs, const __nv_bfloat16* Ks, int r0,
                                       int lane, float scale, int S) {
#pragma unroll
  for (int nt = 0; nt < 8; ++nt)
#pragma unroll
    for (int i = 0; i < 4; ++i) s[nt][i] = 0.f;
#pragma unroll
  for (int kk = 0; kk < kD / 16; ++kk) {
    uint32_t a[4];
    load_a(a, Qs, r0, kk * 16, lane);
#pragma unroll
    for (int nt = 0; nt < 8; nt += 2) {
      uint32_t b[4];
      load_b_nk(b, Ks, nt * 8, kk * 16, lane);
      mma16816(s[nt], a[0], a[1], a[2], a[3], b[0], b[1]);
      mma16816(s[nt + 1], a[0], a[1], a[2], a[3], b[2], b[3]);
    }
  }
  const int c2 = (lane & 3) * 2;
#pragma unroll
  for (int nt = 0; nt < 8; ++nt)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int key = nt * 8 + c2 + (i & 1);
      s[nt][i] = key < S ? s[nt][i] * scale : -INFINITY;
    }
}

__global__ void __launch_bounds__(kThreads) vit_attn_fwd_kernel(const __nv_bfloat16* __restrict__ qkv,
                                                                __nv_bfloat16* __restrict__ out, float* __restrict__ lse,
                                                                int S, int nh, float scale) {
  pdl_begin();
  __shared__ __align__(16) __nv_bfloat16 Qs[kS * kLd], Ks[kS * kLd], Vs[kS * kLd];
  const int b = blockIdx.x / nh, h = blockIdx.x - b * nh;
  const long long row0 = static_cast<long long>(b) * S, ld = 3LL * nh * kD;
  load_tile(Qs, qkv, row0, ld, h * kD, S);
  load_tile(Ks, qkv, row0, ld, (nh + h) * kD, S);
  load_tile(Vs, qkv, row0, ld, (2 * nh + h) * kD, S);
  cp_async_wait_all();
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, r0 = warp * 16;
  if (r0 >= S) return;
  float s[8][4];
  scores(s, Qs, Ks, r0, lane, scale, S);
  // rows g = lane / 4 (values 0, 1) and g + 8 (values 2, 3); a row lives in the 4 lanes of a quad
  float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
    mx0 = fmaxf(mx0, fmaxf(s[nt][0], s[nt][1]));
    mx1 = fmaxf(mx1, fmaxf(s[nt][2], s[nt][3]));
  }
#pragma unroll
  for (int o = 1; o < 4; o <<= 1) {
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
  }
  float sum0 = 0.f, sum1 = 0.f;
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
    s[nt][0] = __expf(s[nt][0] - mx0);
    s[nt][1] = __expf(s[nt][1] - mx0);
    s[nt][2] = __expf(s[nt][2] - mx1);
    s[nt][3] = __expf(s[nt][3] - mx1);
    sum0 += s[nt][0] + s[nt][1];
    sum1 += s[nt][2] + s[nt][3];
  }
#pragma unroll
  for (int o = 1; o < 4; o <<= 1) {
    sum0 += __shfl_xor_sync(0xffffffffu, sum0, o);
    sum1 += __shfl_xor_sync(0xffffffffu, sum1, o);
  }
  // O = P V: the score fragments are the A fragments of the next MMA (k = keys)
  float o[8][4];
#pragma unroll
  for (int dt = 0; dt < 8; ++dt)
#pragma unroll
    for (int i = 0; i < 4; ++i) o[dt][i] = 0.f;
#pragma unroll
  for (int kk = 0; kk < kS / 16; ++kk) {
    const uint32_t a0 = pack2(s[2 * kk][0], s[2 * kk][1]), a1 = pack2(s[2 * kk][2], s[2 * kk][3]);
    const uint32_t a2 = pack2(s[2 * kk + 1][0], s[2 * kk + 1][1]), a3 = pack2(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
    for (int dt = 0; dt < 8; dt += 2) {
      uint32_t bb[4];
      load_b_kn(bb, Vs, dt * 8, kk * 16, lane);
      mma16816(o[dt], a0, a1, a2, a3, bb[0], bb[1]);
      mma16816(o[dt + 1], a0, a1, a2, a3, bb[2], bb[3]);
    }
  }
  const int g = lane >> 2, c2 = (lane & 3) * 2;
  const float inv0 = 1.f / sum0, inv1 = 1.f / sum1;
  const int q0 = r0 + g, q1 = r0 + g + 8;
  const long long ldo = static_cast<long long>(nh) * kD;
#pragma unroll
  for (int dt = 0; dt < 8; ++dt) {
    const int col = h * kD + dt * 8 + c2;
    if (q0 < S)
      *reinterpret_cast<uint32_t*>(out + (row0 + q0) * ldo + col) = pack2(o[dt][0] * inv0, o[dt][1] * inv0);
    if (q1 < S)
      *reinterpret_cast<uint32_t*>(out + (row0 + q1) * ldo + col) = pack2(o[dt][2] * inv1, o[dt][3] * inv1);
  }
  if ((lane & 3) == 0) {
    float* l = lse + (static_cast<long long>(b) * nh + h) * S;
    if (q0 < S) l[q0] = mx0 + __logf(sum0);
    if (q1 < S) l[q1] = mx1 + __logf(sum1);
  }
}

__global__ void __launch_bounds__(kThreads, 4) vit_attn_bwd_kernel(const __nv_bfloat16* qkv,
                                                                const __nv_bfloat16* __restrict__ out,
                                                                const __nv_bfloat16* __restrict__ dout,
                                                                const float* __restrict__ lse, __nv_bfloat16* dqkv,
                                                                float* __restrict__ dbias, int S, int nh,
                                                                float scale) {
  pdl_begin();
  extern __shared__ __align__(16) uint8_t attn_smem[];  // 6 tiles of 64 x 72 bf16 (55 KB) + D: 4 CTAs per SM
  __nv_bfloat16* Qs = reinterpret_cast<__nv_bfloat16*>(attn_smem);
  __nv_bfloat16* Ks = Qs + kS * kLd;
  __nv_bfloat16* Vs = Ks + kS * kLd;
  __nv_bfloat16* dOs = Vs + kS * kLd;
  __nv_bfloat16* Ps = dOs + kS * kLd;
  __nv_bfloat16* dSs = Ps + kS * kLd;
  // column sums over this warp's 16 rows of one 16 x 64 C-fragment block (values rounded to bf16,
  // as a column reduction of the stored gradient would see them) -> dst[col] (float2 atomics into
  // global memory when `atomic`, else plain shared-memory stores)
  auto colsum16 = [&](const float (&v)[8][4], float mul, bool ok0, bool ok1, float* dst, bool atomic) {
    const int lane_ = threadIdx.x & 31;
#pragma unroll
    for (int dt = 0; dt < 8; ++dt) {
      float c0 = (ok0 ? __bfloat162float(__float2bfloat16_rn(v[dt][0] * mul)) : 0.f) +
                 (ok1 ? __bfloat162float(__float2bfloat16_rn(v[dt][2] * mul)) : 0.f);
      float c1 = (ok0 ? __bfloat162float(__float2bfloat16_rn(v[dt][1] * mul)) : 0.f) +
                 (ok1 ? __bfloat162float(__float2bfloat16_rn(v[dt][3] * mul)) : 0.f);
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {  // sum over the 8 row groups (lanes with the same lane % 4)
        c0 += __shfl_xor_sync(0xffffffffu, c0, o);
        c1 += __shfl_xor_sync(0xffffffffu, c1, o);
      }
      if (lane_ < 4) {
        if (atomic) {
          atomicAdd(reinterpret_cast<float2*>(dst + dt * 8 + 2 * lane_), make_float2(c0, c1));
        } else {
          dst[dt * 8 + 2 * lane_] = c0;
          dst[dt * 8 + 2 * lane_ + 1] = c1;
        }
      }
    }
  };
  const int b = blockIdx.x / nh, h = blockIdx.x - b * nh;
  const long long row0 = static_cast<long long>(b) * S, ld = 3LL * nh * kD, ldo = static_cast<long long>(nh) * kD;
  (void)out;  // the flash-attention signature keeps O; D = rowsum(dO * O) is taken as rowsum(P * dP) below
  load_tile(Qs, qkv, row0, ld, h * kD, S);
  load_tile(Ks, qkv, row0, ld, (nh + h) * kD, S);
  load_tile(Vs, qkv, row0, ld, (2 * nh + h) * kD, S);
  load_tile(dOs, dout, row0, ldo, h * kD, S);
  cp_async_wait_all();
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, r0 = warp * 16;
  const int g = lane >> 2, c2 = (lane & 3) * 2;
  // ---- phase 1 (query rows r0..r0+15): P, dP = dO V^T, dS = P (dP - D); dQ = scale dS K
  {
    float s[8][4];
    scores(s, Qs, Ks, r0, lane, scale, S);
    const int q0 = r0 + g, q1 = r0 + g + 8;
    const float* l = lse + (static_cast<long long>(b) * nh + h) * S;
    const float l0 = q0 < S ? l[q0] : 0.f, l1 = q1 < S ? l[q1] : 0.f;
    float dp[8][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) dp[nt][i] = 0.f;
#pragma unroll
    for (int kk = 0; kk < kD / 16; ++kk) {
      uint32_t a[4];
      load_a(a, dOs, r0, kk * 16, lane);
#pragma unroll
      for (int nt = 0; nt < 8; nt += 2) {
        uint32_t bb[4];
        load_b_nk(bb, Vs, nt * 8, kk * 16, lane);
        mma16816(dp[nt], a[0], a[1], a[2], a[3], bb[0], bb[1]);
        mma16816(dp[nt + 1], a[0], a[1], a[2], a[3], bb[2], bb[3]);
      }
    }
    // P, and D[q] = sum_k P[q, k] dP[q, k] (= sum_d dO[q, d] O[q, d]: the whole key range of
    // a row is in this warp's fragments, so D needs no pass over O); a row lives in a lane quad
    float d0 = 0.f, d1 = 0.f;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      // padded query rows get P = 0 (their lse is 0 and scores -inf only for padded keys, so zero them)
      s[nt][0] = q0 < S ? __expf(s[nt][0] - l0) : 0.f;
      s[nt][1] = q0 < S ? __expf(s[nt][1] - l0) : 0.f;
      s[nt][2] = q1 < S ? __expf(s[nt][2] - l1) : 0.f;
      s[nt][3] = q1 < S ? __expf(s[nt][3] - l1) : 0.f;
      d0 += s[nt][0] * dp[nt][0] + s[nt][1] * dp[nt][1];
      d1 += s[nt][2] * dp[nt][2] + s[nt][3] * dp[nt][3];
    }
#pragma unroll
    for (int o = 1; o < 4; o <<= 1) {
      d0 += __shfl_xor_sync(0xffffffffu, d0, o);
      d1 += __shfl_xor_sync(0xffffffffu, d1, o);
    }
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const float p0 = s[nt][0], p1 = s[nt][1], p2 = s[nt][2], p3 = s[nt][3];
      s[nt][0] = p0 * (dp[nt][0] - d0);  // dS
      s[nt][1] = p1 * (dp[nt][1] - d0);
      s[nt][2] = p2 * (dp[nt][2] - d1);
      s[nt][3] = p3 * (dp[nt][3] - d1);
      const int key = nt * 8 + c2;
      *reinterpret_cast<uint32_t*>(Ps + q0 * kLd + key) = pack2(p0, p1);
      *reinterpret_cast<uint32_t*>(Ps + q1 * kLd + key) = pack2(p2, p3);
      *reinterpret_cast<uint32_t*>(dSs + q0 * kLd + key) = pack2(s[nt][0], s[nt][1]);
      *reinterpret_cast<uint32_t*>(dSs + q1 * kLd + key) = pack2(s[nt][2], s[nt][3]);
    }
    // dQ = scale * dS K: A = dS (score fragments, k = keys), B = K stored [key][d] = [k][n]
    float dq[8][4];
#pragma unroll
    for (int dt = 0; dt < 8; ++dt)
#pragma unroll
      for (int i = 0; i < 4; ++i) dq[dt][i] = 0.f;
#pragma unroll
    for (int kk = 0; kk < kS / 16; ++kk) {
      const uint32_t a0 = pack2(s[2 * kk][0], s[2 * kk][1]), a1 = pack2(s[2 * kk][2], s[2 * kk][3]);
      const uint32_t a2 = pack2(s[2 * kk + 1][0], s[2 * kk + 1][1]), a3 = pack2(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
      for (int dt = 0; dt < 8; dt += 2) {
        uint32_t bb[4];
        load_b_kn(bb, Ks, dt * 8, kk * 16, lane);
        mma16816(dq[dt], a0, a1, a2, a3, bb[0], bb[1]);
        mma16816(dq[dt + 1], a0, a1, a2, a3, bb[2], bb[3]);
      }
    }
    if (dbias) colsum16(dq, scale, q0 < S, q1 < S, dbias + h * kD, true);  // the q block of bqkv
    __syncthreads();  // every warp's P / dS rows are in shared memory; Q, K, V, dO reads are done
#pragma unroll
    for (int dt = 0; dt < 8; ++dt) {
      const int col = h * kD + dt * 8 + c2;
      if (q0 < S)
        *reinterpret_cast<uint32_t*>(dqkv + (row0 + q0) * ld + col) = pack2(dq[dt][0] * scale, dq[dt][1] * scale);
      if (q1 < S)
        *reinterpret_cast<uint32_t*>(dqkv + (row0 + q1) * ld + col) = pack2(dq[dt][2] * scale, dq[dt][3] * scale);
    }
  }
  // ---- phase 2 (key rows r0..r0+15): dK = scale dS^T Q, dV = P^T dO
  {
    float dk[8][4], dv[8][4];
#pragma unroll
    for (int dt = 0; dt < 8; ++dt)
#pragma unroll
      for (int i = 0; i < 4; ++i) dk[dt][i] = dv[dt][i] = 0.f;
#pragma unroll
    for (int kk = 0; kk < kS / 16; ++kk) {  // k = queries
      uint32_t ad[4], ap[4];
      load_a_t(ad, dSs, r0, kk * 16, lane);
      load_a_t(ap, Ps, r0, kk * 16, lane);
#pragma unroll
      for (int dt = 0; dt < 8; dt += 2) {
        uint32_t bq[4], bo[4];
        load_b_kn(bq, Qs, dt * 8, kk * 16, lane);
        load_b_kn(bo, dOs, dt * 8, kk * 16, lane);
        mma16816(dk[dt], ad[0], ad[1], ad[2], ad[3], bq[0], bq[1]);
        mma16816(dk[dt + 1], ad[0], ad[1], ad[2], ad[3], bq[2], bq[3]);
        mma16816(dv[dt], ap[0], ap[1], ap[2], ap[3], bo[0], bo[1]);
        mma16816(dv[dt + 1], ap[0], ap[1], ap[2], ap[3], bo[2], bo[3]);
      }
    }
    const int k0 = r0 + g, k1 = r0 + g + 8;
    if (dbias) {
      __syncthreads();  // every warp's P / dS / Q / dO reads are done: the P tile holds the k | v sums
      float* bsum = reinterpret_cast<float*>(Ps);  // [4 warps][128]
      colsum16(dk, scale, k0 < S, k1 < S, bsum + warp * 128, false);
      colsum16(dv, 1.f, k0 < S, k1 < S, bsum + warp * 128 + 64, false);
      __syncthreads();
      if (threadIdx.x < 32) {  // one float4 atomic per 4 columns: k at (nh + h) * 64, v at (2 nh + h) * 64
        const int c = threadIdx.x * 4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const float4 t = *reinterpret_cast<const float4*>(bsum + w * 128 + c);
          v = make_float4(v.x + t.x, v.y + t.y, v.z + t.z, v.w + t.w);
        }
        atomicAdd(reinterpret_cast<float4*>(dbias + (c < 64 ? nh : 2 * nh) * kD + h * kD + (c & 63)), v);
      }
    }
#pragma unroll
    for (int dt = 0; dt < 8; ++dt) {
      const int ck = (nh + h) * kD + dt * 8 + c2, cv = (2 * nh + h) * kD + dt * 8 + c2;
      if (k0 < S) {
        *reinterpret_cast<uint32_t*>(dqkv + (row0 + k0) * ld + ck) = pack2(dk[dt][0] * scale, dk[dt][1] * scale);
        *reinterpret_cast<uint32_t*>(dqkv + (row0 + k0) * ld + cv) = pack2(dv[dt][0], dv[dt][1]);
      }
      if (k1 < S) {
        *reinterpret_cast<uint32_t*>(dqkv + (row0 + k1) * ld + ck) = pack2(dk[dt][2] * scale, dk[dt][3] * scale);
        *reinterpret_cast<uint32_t*>(dqkv + (row0 + k1) * ld + cv) = pack2(dv[dt][2], dv[dt][3]);
      }
    }
  }
}

}  // namespace

int launch_vit_attn_fwd(const __nv_bfloat16* qkv, __nv_bfloat16* out, float* lse, int B, int S, int nh, int hd,
                        float scale, cudaStream_t s) {
  if (S < 1 || S > kS || hd != kD || B < 1 || nh < 1) return PF_ERR_INVALID;
  launch_k(vit_attn_fwd_kernel, dim3(B * nh), dim3(kThreads), 0, s, qkv, out, lse, S, nh, scale);
  return status();
}

int launch_vit_attn_bwd(const __nv_bfloat16* qkv, const __nv_bfloat16* out, const __nv_bfloat16* dout,
                        const float* lse, __nv_bfloat16* dqkv, float* dbias, int B, int S, int nh, int hd, float scale,
                        cudaStream_t s) {
  if (S < 1 || S > kS || hd != kD || B < 1 || nh < 1) return PF_ERR_INVALID;
  if (reinterpret_cast<uintptr_t>(dbias) % 16) return PF_ERR_INVALID;  // float4 atomics
  constexpr int smem = 6 * kS * kLd * 2;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(vit_attn_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return PF_ERR_CUDA;
    attr = true;
  }
  launch_k(vit_attn_bwd_kernel, dim3(B * nh), dim3(kThreads), smem, s, qkv, out, dout, lse, dqkv, dbias, S, nh, scale);
  return status();
}

}  // namespace pf
