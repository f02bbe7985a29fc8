// K7 glue of the ViT encoder stage (ViT-L/32): LayerNorm with
// bias, GELU (erf form), per-column bias gradients, the patch / cls / position
// embedding, the cls-row gather for the classification head, and the synthetic
// patch input. All HBM-bound elementwise or row/column reductions over bf16
// activations with fp32 statistics and fp32 parameter gradients.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "kernel_util.cuh"
#include "ptx.cuh"
#include "vit_kernels.cuh"

namespace pf {

namespace {

// LayerNorm forward, one warp per row: mean, then variance around it (second pass
// from L1/L2), y = (x - mean) * rstd * g + b.
__global__ void __launch_bounds__(kBlock) layernorm_fwd_kernel(const __nv_bfloat16* __restrict__ x,
                                                               const __nv_bfloat16* __restrict__ g,
                                                               const __nv_bfloat16* __restrict__ b,
                                                               __nv_bfloat16* __restrict__ y,
                                                               float* __restrict__ mean_out,
                                                               float* __restrict__ rstd_out, int T, int h,
                                                               float eps) {
  pdl_begin();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int t = blockIdx.x * (kBlock / 32) + warp; t < T; t += gridDim.x * (kBlock / 32)) {
    const __nv_bfloat16* xr = x + static_cast<long long>(t) * h;
    float s = 0.f;
    for (int c = lane * 8; c < h; c += 256) {
      float f[8];
      load8(xr + c, f);
#pragma unroll
      for (int i = 0; i < 8; ++i) s += f[i];
    }
    const float mu = warp_sum(s) / h;
    float ss = 0.f;
    for (int c = lane * 8; c < h; c += 256) {
      float f[8];
      load8(xr + c, f);
#pragma unroll
      for (int i = 0; i < 8; ++i) ss += (f[i] - mu) * (f[i] - mu);
    }
    const float r = rsqrtf(warp_sum(ss) / h + eps);
    if (lane == 0) {
      mean_out[t] = mu;
      rstd_out[t] = r;
    }
    __nv_bfloat16* yr = y + static_cast<long long>(t) * h;
    for (int c = lane * 8; c < h; c += 256) {
      float f[8], gg[8], bb[8];
      load8(xr + c, f);
      load8(g + c, gg);
      load8(b + c, bb);
#pragma unroll
      for (int i = 0; i < 8; ++i) f[i] = (f[i] - mu) * r * gg[i] + bb[i];
      store8(yr + c, f);
    }
  }
}

// dx = residual + rstd * (g*dy - mean(g*dy) - xhat * mean(g*dy*xhat)); one warp per row
__global__ void __launch_bounds__(kBlock) layernorm_bwd_kernel(const __nv_bfloat16* __restrict__ x,
                                                               const __nv_bfloat16* __restrict__ g,
                                                               const float* __restrict__ mean,
                                                               const float* __restrict__ rstd,
                                                               const __nv_bfloat16* __restrict__ dy,
                                                               const __nv_bfloat16* __restrict__ residual,
                                                               __nv_bfloat16* __restrict__ dx, int T, int h) {
  pdl_begin();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int t = blockIdx.x * (kBlock / 32) + warp; t < T; t += gridDim.x * (kBlock / 32)) {
    const long long off = static_cast<long long>(t) * h;
    const float mu = mean[t], r = rstd[t];
    float s1 = 0.f, s2 = 0.f;
    for (int c = lane * 8; c < h; c += 256) {
      float xv[8], gv[8], dv[8];
      load8(x + off + c, xv);
      load8(g + c, gv);
      load8(dy + off + c, dv);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float gd = gv[i] * dv[i];
        s1 += gd;
        s2 += gd * (xv[i] - mu) * r;
      }
    }
    const float m1 = warp_sum(s1) / h, m2 = warp_sum(s2) / h;
    for (int c = lane * 8; c < h; c += 256) {
      float xv[8], gv[8], dv[8], out[8];
      load8(x + off + c, xv);
      load8(g + c, gv);
      load8(dy + off + c, dv);
      if (residual) load8(residual + off + c, out);
#pragma unroll
      for (int i = 0; i < 8; ++i)
        out[i] = (residual ? out[i] : 0.f) + r * (gv[i] * dv[i] - m1 - (xv[i] - mu) * r * m2);
      store8(dx + off + c, out);
    }
  }
}

// Row-in-registers LayerNorm for h = 256 * CH: one warp per row, lane holds columns
// lane*8 + 256 j; mean and variance from the registers, x read from HBM once.
template <int CH>
__global__ void __launch_bounds__(kBlock) layernorm_fwd_reg_kernel(const __nv_bfloat16* __restrict__ x,
                                                                   const __nv_bfloat16* __restrict__ g,
                                                                   const __nv_bfloat16* __restrict__ b,
                                                                   __nv_bfloat16* __restrict__ y,
                                                                   float* __restrict__ mean_out,
                                                                   float* __restrict__ rstd_out, int T, float eps) {
  pdl_begin();
  constexpr int H = 256 * CH;
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < T; t += nw) {
    const long long off = static_cast<long long>(t) * H + lane * 8;
    float f[CH][8];
    uint4 gr[CH], br[CH];  // g and b ride with x: their loads do not wait behind the row reductions
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      load8(x + off + 256 * j, f[j]);
      gr[j] = *reinterpret_cast<const uint4*>(g + lane * 8 + 256 * j);
      br[j] = *reinterpret_cast<const uint4*>(b + lane * 8 + 256 * j);
    }
    float sm = 0.f;
#pragma unroll
    for (int j = 0; j < CH; ++j)
#pragma unroll
      for (int i = 0; i < 8; ++i) sm += f[j][i];
    const float mu = warp_sum(sm) / H;
    float ss = 0.f;
#pragma unroll
    for (int j = 0; j < CH; ++j)
#pragma unroll
      for (int i = 0; i < 8; ++i) ss += (f[j][i] - mu) * (f[j][i] - mu);
    const float r = rsqrtf(warp_sum(ss) / H + eps);
    if (lane == 0) {
      mean_out[t] = mu;
      rstd_out[t] = r;
    }
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      float gg[8], bb[8], o[8];
      const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gr[j]);
      const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&br[j]);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 gf = __bfloat1622float2(g2[i]), bf = __bfloat1622float2(b2[i]);
        gg[2 * i] = gf.x;
        gg[2 * i + 1] = gf.y;
        bb[2 * i] = bf.x;
        bb[2 * i + 1] = bf.y;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = (f[j][i] - mu) * r * gg[i] + bb[i];
      store8(y + off + 256 * j, o);
    }
  }
}

// Fused LayerNorm backward for h = 256 * CH, one pass over x and dy:
//   dx = residual + rstd * (g*dy - mean(g*dy) - xhat * mean(g*dy*xhat))
//   dg += sum_t dy * xhat,  db += sum_t dy,  dsum += sum_t dx   (dsum: the bias gradient of the
//   linear layer whose output gradient dx is; nullptr skips it)
// x, dy and the residual of a row are loaded together (one memory round trip per row). Per-lane
// register partials, summed over the block's warps in shared memory, added to the
// fp32 gradients with float4 atomics (one per 4 columns per block).
template <int CH>
__global__ void __launch_bounds__(kBlock, 1) layernorm_bwd_fused_kernel(
    const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ g, const float* __restrict__ mean,
    const float* __restrict__ rstd, const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ residual,
    __nv_bfloat16* __restrict__ dx, float* __restrict__ dg, float* __restrict__ db, float* __restrict__ dsum, int T) {
  pdl_begin();
  constexpr int H = 256 * CH;
  constexpr int NW = kBlock / 32;
  extern __shared__ float red[];  // [3][NW][H]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float ag[CH * 8], ab[CH * 8], as[CH * 8];
#pragma unroll
  for (int i = 0; i < CH * 8; ++i) ag[i] = ab[i] = as[i] = 0.f;
  for (int t = blockIdx.x * NW + warp; t < T; t += gridDim.x * NW) {
    const long long off = static_cast<long long>(t) * H + lane * 8;
    const float mu = mean[t], r = rstd[t];
    float xv[CH][8], dv[CH][8];
    uint4 rr[CH];
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      load8(x + off + 256 * j, xv[j]);
      load8(dy + off + 256 * j, dv[j]);
      if (residual) rr[j] = *reinterpret_cast<const uint4*>(residual + off + 256 * j);
    }
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      float gv[8];
      load8(g + lane * 8 + 256 * j, gv);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float gd = gv[i] * dv[j][i];
        s1 += gd;
        s2 += gd * (xv[j][i] - mu) * r;
      }
    }
    const float m1 = warp_sum(s1) / H, m2 = warp_sum(s2) / H;
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      float gv[8], out[8];
      load8(g + lane * 8 + 256 * j, gv);
      if (residual) {
        const __nv_bfloat162* r2 = reinterpret_cast<const __nv_bfloat162*>(&rr[j]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 t2 = __bfloat1622float2(r2[i]);
          out[2 * i] = t2.x;
          out[2 * i + 1] = t2.y;
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float xh = (xv[j][i] - mu) * r;
        out[i] = (residual ? out[i] : 0.f) + r * (gv[i] * dv[j][i] - m1 - xh * m2);
        ag[8 * j + i] += dv[j][i] * xh;
        ab[8 * j + i] += dv[j][i];
      }
      store8(dx + off + 256 * j, out);
      if (dsum) {  // the bias gradient sums the stored (bf16-rounded) dx, as a column reduction of dx would
#pragma unroll
        for (int i = 0; i < 8; ++i) as[8 * j + i] += __bfloat162float(__float2bfloat16_rn(out[i]));
      }
    }
  }
  auto park = [&](const float (&acc)[CH * 8], int a) {
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      float* slot = red + (a * NW + warp) * H + lane * 8 + 256 * j;
      reinterpret_cast<float4*>(slot)[0] = make_float4(acc[8 * j], acc[8 * j + 1], acc[8 * j + 2], acc[8 * j + 3]);
      reinterpret_cast<float4*>(slot)[1] =
          make_float4(acc[8 * j + 4], acc[8 * j + 5], acc[8 * j + 6], acc[8 * j + 7]);
    }
  };
  auto flush = [&](float* outp, int a) {
    for (int c = threadIdx.x * 4; c < H; c += kBlock * 4) {
      float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const float4 v = *reinterpret_cast<const float4*>(red + (a * NW + w) * H + c);
        sum = make_float4(sum.x + v.x, sum.y + v.y, sum.z + v.z, sum.w + v.w);
      }
      atomicAdd(reinterpret_cast<float4*>(outp + c), sum);
    }
  };
  if (dg) park(ag, 0);
  if (db) park(ab, 1);
  if (dsum) park(as, 2);
  __syncthreads();
  if (dg) flush(dg, 0);
  if (db) flush(db, 1);
  if (dsum) flush(dsum, 2);
}

// Column reductions over T rows (block = 32 column groups of 8 x 8 row lanes):
//   dg[c] += sum_t dy[t,c] * (x[t,c] - mean[t]) * rstd[t]   (when x != nullptr)
//   db[c] += sum_t dy[t,c]
__global__ void __launch_bounds__(kBlock) column_reduce_kernel(const __nv_bfloat16* __restrict__ dy, long long ldy,
                                                               const __nv_bfloat16* __restrict__ x,
                                                               const float* __restrict__ mean,
                                                               const float* __restrict__ rstd,
                                                               float* __restrict__ dg, float* __restrict__ db,
                                                               int T, int n, int rows_per_block) {
  pdl_begin();
  __shared__ float pg[8][256 + 4];
  __shared__ float pb[8][256 + 4];
  const int cg = threadIdx.x & 31, rl = threadIdx.x >> 5;
  const int c = blockIdx.x * 256 + cg * 8;
  const int r0 = blockIdx.y * rows_per_block;
  const int r1 = min(T, r0 + rows_per_block);
  float ag[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  float ab[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (c < n) {
    for (int t = r0 + rl; t < r1; t += 8) {
      float dv[8];
      load8(dy + static_cast<long long>(t) * ldy + c, dv);
#pragma unroll
      for (int i = 0; i < 8; ++i) ab[i] += dv[i];
      if (x) {
        float xv[8];
        load8(x + static_cast<long long>(t) * n + c, xv);
        const float mu = mean[t], r = rstd[t];
#pragma unroll
        for (int i = 0; i < 8; ++i) ag[i] += dv[i] * (xv[i] - mu) * r;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    pg[rl][cg * 8 + i] = ag[i];
    pb[rl][cg * 8 + i] = ab[i];
  }
  __syncthreads();
  const int col = blockIdx.x * 256 + threadIdx.x;
  if (col < n) {
    float sg = 0.f, sb = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      sg += pg[k][threadIdx.x];
      sb += pb[k][threadIdx.x];
    }
    if (x && dg) atomicAdd(&dg[col], sg);
    if (db) atomicAdd(&db[col], sb);
  }
}


__global__ void gelu_fwd_kernel(const __nv_bfloat16* __restrict__ pre, __nv_bfloat16* __restrict__ act, long long n8) {
  pdl_begin();
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n8;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    float f[8];
    load8(pre + i * 8, f);
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
      const float2 g = gelu_erf2(make_float2(f[k], f[k + 1]));
      f[k] = g.x;
      f[k + 1] = g.y;
    }
    store8(act + i * 8, f);
  }
}

__global__ void gelu_bwd_kernel(const __nv_bfloat16* __restrict__ pre, const __nv_bfloat16* __restrict__ dact,
                                __nv_bfloat16* __restrict__ dpre, long long n8) {
  pdl_begin();
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n8;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    float p[8], d[8];
    load8(pre + i * 8, p);
    load8(dact + i * 8, d);
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
      const float2 g = mul2(make_float2(d[k], d[k + 1]), gelu_erf_grad2(make_float2(p[k], p[k + 1])));
      d[k] = g.x;
      d[k + 1] = g.y;
    }
    store8(dpre + i * 8, d);
  }
}

__global__ void add_bias_kernel(__nv_bfloat16* __restrict__ c, long long ldc, const __nv_bfloat16* __restrict__ bias,
                                int M, int N) {
  pdl_begin();
  const int chunks = N / 8;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < static_cast<long long>(M) * chunks;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = i / chunks;
    const int col = static_cast<int>(i - r * chunks) * 8;
    float v[8], b[8];
    load8(c + r * ldc + col, v);
    load8(bias + col, b);
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] += b[k];
    store8(c + r * ldc + col, v);
  }
}

// x[b, 0] = cls + pos[0]; x[b, 1 + p] = E[b * np + p] + patch_bias + pos[1 + p]
__global__ void vit_embed_fwd_kernel(const __nv_bfloat16* __restrict__ E, const __nv_bfloat16* __restrict__ pbias,
                                     const __nv_bfloat16* __restrict__ cls, const __nv_bfloat16* __restrict__ pos,
                                     __nv_bfloat16* __restrict__ x, int B, int S, int h) {
  pdl_begin();
  const int chunks = h / 8;
  const long long total = static_cast<long long>(B) * S * chunks;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long row = i / chunks;
    const int c = static_cast<int>(i - row * chunks) * 8;
    const int b = static_cast<int>(row / S), p = static_cast<int>(row - static_cast<long long>(b) * S);
    float v[8], q[8];
    load8(pos + static_cast<long long>(p) * h + c, q);
    if (p == 0) {
      load8(cls + c, v);
    } else {
      float bb[8];
      load8(E + (static_cast<long long>(b) * (S - 1) + (p - 1)) * h + c, v);
      load8(pbias + c, bb);
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] += bb[k];
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] += q[k];
    store8(x + row * h + c, v);
  }
}

// Backward of vit_embed_fwd: dE rows gathered from dx, dpos[p] += sum_b dx[b, p],
// dcls += sum_b dx[b, 0], dpatch_bias += sum_b sum_{p>0} dx[b, p].
__global__ void vit_embed_bwd_kernel(const __nv_bfloat16* __restrict__ dx, __nv_bfloat16* __restrict__ dE,
                                     float* __restrict__ dpos, float* __restrict__ dcls, float* __restrict__ dpbias,
                                     int B, int S, int h) {
  pdl_begin();
  const int chunks = h / 8;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
       i < static_cast<long long>(S) * chunks; i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int p = static_cast<int>(i / chunks);
    const int c = static_cast<int>(i - static_cast<long long>(p) * chunks) * 8;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int b = 0; b < B; ++b) {
      const long long row = static_cast<long long>(b) * S + p;
      float v[8];
      load8(dx + row * h + c, v);
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] += v[k];
      if (p > 0) *reinterpret_cast<uint4*>(dE + (static_cast<long long>(b) * (S - 1) + (p - 1)) * h + c) =
          *reinterpret_cast<const uint4*>(dx + row * h + c);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      dpos[static_cast<long long>(p) * h + c + k] += acc[k];
      if (p == 0) dcls[c + k] += acc[k];
      else atomicAdd(&dpbias[c + k], acc[k]);
    }
  }
}

// out[b] = x[b * S + row_in_seq]   (cls rows for the head) / scatter back into zeros
__global__ void gather_rows_kernel(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ out, int B,
                                   int S, int h) {
  pdl_begin();
  const int chunks = h / 8;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
       i < static_cast<long long>(B) * chunks; i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long b = i / chunks;
    const int c = static_cast<int>(i - b * chunks) * 8;
    *reinterpret_cast<uint4*>(out + b * h + c) = *reinterpret_cast<const uint4*>(x + b * S * h + c);
  }
}

__global__ void scatter_rows_kernel(const __nv_bfloat16* __restrict__ src, __nv_bfloat16* __restrict__ dx, int B,
                                    int S, int h) {
  pdl_begin();
  const int chunks = h / 8;
  const long long total = static_cast<long long>(B) * S * chunks;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long row = i / chunks;
    const int c = static_cast<int>(i - row * chunks) * 8;
    const long long b = row / S;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (row - b * S == 0) v = *reinterpret_cast<const uint4*>(src + b * h + c);
    *reinterpret_cast<uint4*>(dx + row * h + c) = v;
  }
}

// deterministic synthetic pixels in [-1, 1) (splitmix64 of the element index)
__global__ void synthetic_patches_kernel(__nv_bfloat16* __restrict__ out, long long n, uint64_t seed) {
  pdl_begin();
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    uint64_t z = seed + static_cast<uint64_t>(i + 1) * 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    z ^= z >> 31;
    out[i] = __float2bfloat16_rn(static_cast<float>(z >> 40) * 0x1.0p-23f - 1.f);
  }
}

void column_grid(int T, int n, int* col_blocks, int* row_chunks, int* rows_per_block) {
  *col_blocks = (n + 255) / 256;
  int rc = std::max(1, (2 * num_sms()) / *col_blocks);
  *rows_per_block = std::max(8, (T + rc - 1) / rc);
  *row_chunks = (T + *rows_per_block - 1) / *rows_per_block;
}

}  // namespace

int launch_layernorm_fwd(const __nv_bfloat16* x, const __nv_bfloat16* g, const __nv_bfloat16* b, __nv_bfloat16* y,
                         float* mean, float* rstd, int T, int h, float eps, cudaStream_t s) {
  if (h % 8) return PF_ERR_INVALID;
  const dim3 grid(grid_for((T + 7) / 8));
  switch (h) {
    case 256: launch_k(layernorm_fwd_reg_kernel<1>, grid, dim3(kBlock), 0, s, x, g, b, y, mean, rstd, T, eps); return status();
    case 512: launch_k(layernorm_fwd_reg_kernel<2>, grid, dim3(kBlock), 0, s, x, g, b, y, mean, rstd, T, eps); return status();
    case 1024: launch_k(layernorm_fwd_reg_kernel<4>, grid, dim3(kBlock), 0, s, x, g, b, y, mean, rstd, T, eps); return status();
    default: break;
  }
  launch_k(layernorm_fwd_kernel, grid, dim3(kBlock), 0, s, x, g, b, y, mean, rstd, T, h, eps);
  return status();
}

namespace {
template <int CH>
int launch_layernorm_bwd_fused(const __nv_bfloat16* x, const __nv_bfloat16* g, const float* mean, const float* rstd,
                               const __nv_bfloat16* dy, const __nv_bfloat16* residual, __nv_bfloat16* dx, float* dg,
                               float* db, float* dsum, int T, cudaStream_t s) {
  constexpr int smem = 3 * (kBlock / 32) * 256 * CH * 4;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(layernorm_bwd_fused_kernel<CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
        cudaSuccess)
      return PF_ERR_CUDA;
    attr = true;
  }
  const int grid = std::max(1, std::min(num_sms(), (T + 7) / 8));
  launch_k(layernorm_bwd_fused_kernel<CH>, dim3(grid), dim3(kBlock), smem, s, x, g, mean, rstd, dy, residual, dx, dg,
           db, dsum, T);
  return status();
}
}  // namespace

int launch_layernorm_bwd(const __nv_bfloat16* x, const __nv_bfloat16* g, const float* mean, const float* rstd,
                         const __nv_bfloat16* dy, const __nv_bfloat16* residual, __nv_bfloat16* dx, float* dg,
                         float* db, float* dsum, int T, int h, cudaStream_t s) {
  if (h % 8) return PF_ERR_INVALID;
  switch (h) {
    case 256: return launch_layernorm_bwd_fused<1>(x, g, mean, rstd, dy, residual, dx, dg, db, dsum, T, s);
    case 512: return launch_layernorm_bwd_fused<2>(x, g, mean, rstd, dy, residual, dx, dg, db, dsum, T, s);
    case 1024: return launch_layernorm_bwd_fused<4>(x, g, mean, rstd, dy, residual, dx, dg, db, dsum, T, s);
    default: break;
  }
  launch_k(layernorm_bwd_kernel, dim3(grid_for((T + 7) / 8)), dim3(kBlock), 0, s, x, g, mean, rstd, dy, residual, dx, T, h);
  int rc = status();
  if (rc == PF_OK && (dg || db)) {
    int cb, rcn, rpb;
    column_grid(T, h, &cb, &rcn, &rpb);
    launch_k(column_reduce_kernel, dim3(dim3(cb, rcn)), dim3(kBlock), 0, s, dy, h, x, mean, rstd, dg, db, T, h, rpb);
    rc = status();
  }
  if (rc == PF_OK && dsum) rc = launch_bias_grad(dx, h, dsum, T, h, s);
  return rc;
}

int launch_bias_grad(const __nv_bfloat16* dy, long long ldy, float* db, int T, int n, cudaStream_t s) {
  if (n % 8 || ldy % 8) return PF_ERR_INVALID;
  int cb, rcn, rpb;
  column_grid(T, n, &cb, &rcn, &rpb);
  launch_k(column_reduce_kernel, dim3(dim3(cb, rcn)), dim3(kBlock), 0, s, dy, ldy, nullptr, nullptr, nullptr, nullptr, db, T, n, rpb);
  return status();
}

int launch_gelu_fwd(const __nv_bfloat16* pre, __nv_bfloat16* act, long long n, cudaStream_t s) {
  if (n % 8) return PF_ERR_INVALID;
  launch_k(gelu_fwd_kernel, dim3(grid_for((n / 8 + kBlock - 1) / kBlock)), dim3(kBlock), 0, s, pre, act, n / 8);
  return status();
}

int launch_gelu_bwd(const __nv_bfloat16* pre, const __nv_bfloat16* dact, __nv_bfloat16* dpre, long long n,
                    cudaStream_t s) {
  if (n % 8) return PF_ERR_INVALID;
  launch_k(gelu_bwd_kernel, dim3(grid_for((n / 8 + kBlock - 1) / kBlock)), dim3(kBlock), 0, s, pre, dact, dpre, n / 8);
  return status();
}

int launch_add_bias(__nv_bfloat16* c, long long ldc, const __nv_bfloat16* bias, int M, int N, cudaStream_t s) {
  if (N % 8 || ldc % 8) return PF_ERR_INVALID;
  launch_k(add_bias_kernel, dim3(grid_for((static_cast<long long>(M) * (N / 8) + kBlock - 1) / kBlock)), dim3(kBlock), 0, s, c, ldc, bias,
                                                                                                           M, N);
  return status();
}

int launch_vit_embed_fwd(const __nv_bfloat16* E, const __nv_bfloat16* pbias, const __nv_bfloat16* cls,
                         const __nv_bfloat16* pos, __nv_bfloat16* x, int B, int S, int h, cudaStream_t s) {
  if (h % 8) return PF_ERR_INVALID;
  launch_k(vit_embed_fwd_kernel, dim3(grid_for((static_cast<long long>(B) * S * (h / 8) + kBlock - 1) / kBlock)), dim3(kBlock), 0, s, 
      E, pbias, cls, pos, x, B, S, h);
  return status();
}

int launch_vit_embed_bwd(const __nv_bfloat16* dx, __nv_bfloat16* dE, float* dpos, float* dcls, float* dpbias, int B,
                         int S, int h, cudaStream_t s) {
  if (h % 8) return PF_ERR_INVALID;
  launch_k(vit_embed_bwd_kernel, dim3(grid_for((static_cast<long long>(S) * (h / 8) + kBlock - 1) / kBlock)), dim3(kBlock), 0, s, 
      dx, dE, dpos, dcls, dpbias, B, S, h);
  return status();
}

int launch_gather_rows(const __nv_bfloat16* x, __nv_bfloat16* out, int B, int S, int h, cudaStream_t s) {
  if (h % 8) return PF_ERR_INVALID;
  launch_k(gather_rows_kernel, dim3(grid_for((static_cast<long long>(B) * (h / 8) + kBlock - 1) / kBlock)), dim3(kBlock), 0, s, x, out, B,
                                                                                                              S, h);
  return status();
}

int launch_scatter_rows(const __nv_bfloat16* src, __nv_bfloat16* dx, int B, int S, int h, cudaStream_t s) {
  if (h % 8) return PF_ERR_INVALID;
  launch_k(scatter_rows_kernel, dim3(grid_for((static_cast<long long>(B) * S * (h / 8) + kBlock - 1) / kBlock)), dim3(kBlock), 0, s, 
      src, dx, B, S, h);
  return status();
}

int launch_synthetic_patches(__nv_bfloat16* out, long long n, uint64_t seed, cudaStream_t s) {
  launch_k(synthetic_patches_kernel, dim3(grid_for((n + kBlock - 1) / kBlock)), dim3(kBlock), 0, s, out, n, seed);
  return status();
}

}  // namespace pf
