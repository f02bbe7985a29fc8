// Memory-bound sm_100a kernels of the stage step:
//   K4  APF freeze metric (standalone and fused into the optimizer)
//   K5  frozen-unit bitmask -> per-matrix work lists for the masked dW GEMM
//   K6  masked SGD step over 128x128 units (skips units frozen in every microbatch)
//   K7  LLaMA glue: embedding, RMSNorm, RoPE, SwiGLU, fused cross-entropy, init
// All loads/stores are 16-byte vectorised and coalesced along rows; grids are
// sized as multiples of the SM count (persistent grid-stride loops).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstdint>

#include "kernels.cuh"
#include "kernel_util.cuh"
#include "ptx.cuh"
#include "pf_device_internal.hpp"

namespace pf {

namespace {

__device__ __forceinline__ const UnitMatrix& find_matrix(const UnitMatrix* mats, int nmats, int u) {
  int lo = 0, hi = nmats - 1;
  while (lo < hi) {  // last matrix with unit_offset <= u
    const int mid = (lo + hi + 1) >> 1;
    if (mats[mid].unit_offset <= u) lo = mid;
    else hi = mid - 1;
  }
  return mats[lo];
}

// ------------------------------------------------------------------ K5
__global__ void __launch_bounds__(kBlock) mask_to_lists_kernel(const uint64_t* __restrict__ words,
                                                               const UnitMatrix* __restrict__ mats,
                                                               int* __restrict__ lists, int* __restrict__ counts) {
  pdl_begin();
  const UnitMatrix m = mats[blockIdx.x];
  __shared__ int warp_tot[kBlock / 32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // each thread owns 32 consecutive units of the chunk
  for (int chunk = 0; chunk < m.units; chunk += kBlock * 32) {
    const int first = chunk + threadIdx.x * 32;
    uint32_t unfrozen = 0;
    if (first < m.units) {
      const long long g = static_cast<long long>(m.unit_offset) + first;  // global unit id
      const uint64_t w0 = words[g >> 6];
      const uint64_t w1 = ((g & 63) != 0) ? words[(g >> 6) + 1] : 0;  // may read one word past a segment; buffer is padded
      const uint64_t bits = (g & 63) ? ((w0 >> (g & 63)) | (w1 << (64 - (g & 63)))) : w0;
      unfrozen = ~static_cast<uint32_t>(bits);
      const int valid = m.units - first;
      if (valid < 32) unfrozen &= (1u << valid) - 1u;
    }
    const int cnt = __popc(unfrozen);
    // block exclusive scan of cnt
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    int warp_base = 0;
    for (int w = 0; w < warp; ++w) warp_base += warp_tot[w];
    int pos = carry + warp_base + incl - cnt;
    int* out = lists + m.unit_offset;
    for (uint32_t b = unfrozen; b; b &= b - 1) out[pos++] = first + __ffs(b) - 1;
    __syncthreads();
    if (threadIdx.x == kBlock - 1) carry += warp_base + incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) counts[blockIdx.x] = carry;
}

// ------------------------------------------------------------------ K5p
// One block per matrix; warp w walks groups w, w + 8, ...: a ballot over 32 row
// blocks at a time finds the group's unfrozen units, its padded count goes to
// shared memory, a block scan gives every group its even base, and a second
// ballot pass writes the ids.
__global__ void __launch_bounds__(kBlock) mask_to_pairs_kernel(const uint64_t* __restrict__ words,
                                                               const UnitMatrix* __restrict__ mats,
                                                               int* __restrict__ pairs, int* __restrict__ counts) {
  pdl_begin();
  const UnitMatrix m = mats[blockIdx.x];
  __shared__ int base[kPairGroups + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tiles_n = m.tiles_n, tiles_m = m.units / m.tiles_n;
  const int band = pair_band_rows(tiles_m, tiles_n);
  const int groups = pair_groups(tiles_m, tiles_n);
  auto unfrozen = [&](int mb, int nb, int mb_end) -> bool {
    if (mb >= mb_end) return false;
    const long long g = static_cast<long long>(m.unit_offset) + static_cast<long long>(mb) * tiles_n + nb;
    return ((words[g >> 6] >> (g & 63)) & 1ull) == 0;
  };
  for (int g = warp; g < groups; g += kBlock / 32) {
    const int b = g / tiles_n, nb = g - b * tiles_n;
    const int mb0 = b * band, mb1 = min(tiles_m, mb0 + band);
    int cnt = 0;
    for (int r0 = mb0; r0 < mb1; r0 += 32) cnt += __popc(__ballot_sync(0xffffffffu, unfrozen(r0 + lane, nb, mb1)));
    if (lane == 0) base[g + 1] = cnt + (cnt & 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    base[0] = 0;
    for (int g = 0; g < groups; ++g) base[g + 1] += base[g];
    counts[blockIdx.x] = base[groups];
  }
  __syncthreads();
  int* out = pairs + m.pair_offset;
  for (int g = warp; g < groups; g += kBlock / 32) {
    const int b = g / tiles_n, nb = g - b * tiles_n;
    const int mb0 = b * band, mb1 = min(tiles_m, mb0 + band);
    int pos = base[g];
    for (int r0 = mb0; r0 < mb1; r0 += 32) {
      const bool u = unfrozen(r0 + lane, nb, mb1);
      const uint32_t bal = __ballot_sync(0xffffffffu, u);
      if (u) out[pos + __popc(bal & ((1u << lane) - 1u))] = (r0 + lane) * tiles_n + nb;
      pos += __popc(bal);
    }
    if (lane == 0 && pos < base[g + 1]) out[pos] = -1;
  }
}

// ------------------------------------------------------------------ K5r
// One block of 1024 threads per matrix, one thread per unit row: the row's frozen bits are
// read 64 at a time (two words and a funnel shift), the unfrozen count goes to shared memory,
// a block scan gives each row its entry base, and the thread then walks its row's unfrozen
// units in order writing pairs (a row with an odd count ends with {u, -1}).
constexpr int kRowPairRows = 4096;
constexpr int kRowPairThreads = 1024;
__device__ __forceinline__ uint64_t bits64(const uint64_t* __restrict__ words, long long start) {
  const uint64_t w0 = words[start >> 6];
  const int sh = static_cast<int>(start & 63);
  return sh ? (w0 >> sh) | (words[(start >> 6) + 1] << (64 - sh)) : w0;  // buffer padded by one word
}
__global__ void __launch_bounds__(kRowPairThreads) mask_to_rowpairs_kernel(const uint64_t* __restrict__ words,
                                                                           const UnitMatrix* __restrict__ mats,
                                                                           int* __restrict__ lists,
                                                                           int* __restrict__ counts) {
  pdl_begin();
  const UnitMatrix m = mats[blockIdx.x];
  __shared__ int base[kRowPairRows + 1];
  __shared__ int warp_tot[kRowPairThreads / 32];
  const int tiles_n = m.tiles_n, tiles_m = m.units / m.tiles_n;
  auto row_unfrozen = [&](int mb, int c0) -> uint64_t {  // unfrozen mask of columns [c0, c0 + 64)
    const uint64_t f = bits64(words, static_cast<long long>(m.unit_offset) + static_cast<long long>(mb) * tiles_n + c0);
    const int valid = tiles_n - c0;
    return ~f & (valid >= 64 ? ~0ull : ((1ull << valid) - 1ull));
  };
  for (int mb = threadIdx.x; mb < tiles_m; mb += kRowPairThreads) {
    int cnt = 0;
    for (int c0 = 0; c0 < tiles_n; c0 += 64) cnt += __popcll(row_unfrozen(mb, c0));
    base[mb + 1] = (cnt + 1) >> 1;
  }
  __syncthreads();
  // block-wide exclusive scan of base[1..tiles_m] (chunks of kRowPairThreads rows)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int carry = 0;
  for (int r0 = 0; r0 < tiles_m; r0 += kRowPairThreads) {
    const int r = r0 + threadIdx.x;
    const int v = r < tiles_m ? base[r + 1] : 0;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    int wbase = 0;
    for (int w = 0; w < warp; ++w) wbase += warp_tot[w];
    int blk = 0;
    for (int w = 0; w < kRowPairThreads / 32; ++w) blk += warp_tot[w];
    __syncthreads();
    if (r < tiles_m) base[r + 1] = carry + wbase + incl;
    carry += blk;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    base[0] = 0;
    counts[blockIdx.x] = base[tiles_m];
  }
  __syncthreads();
  int2* out = reinterpret_cast<int2*>(lists + m.pair_offset);
  for (int mb = threadIdx.x; mb < tiles_m; mb += kRowPairThreads) {
    int e = base[mb], pending = -1;
    for (int c0 = 0; c0 < tiles_n; c0 += 64) {
      for (uint64_t b = row_unfrozen(mb, c0); b; b &= b - 1) {
        const int u = mb * tiles_n + c0 + __ffsll(static_cast<long long>(b)) - 1;
        if (pending < 0) {
          pending = u;
        } else {
          out[e++] = make_int2(pending, u);
          pending = -1;
        }
      }
    }
    if (pending >= 0) out[e] = make_int2(pending, -1);
  }
}

// ------------------------------------------------------------------ K6 (+K4 fused)
struct AdamCoef {
  float step_size;  // lr / bc1
  float rsqrt_bc2;  // 1 / sqrt(bc2)
  float decay;      // 1 - lr * weight_decay
};

__device__ __forceinline__ AdamCoef adam_coef(const OptimArgs& a, int k) {
  const double bc1 = 1.0 - pow(a.beta1_d, static_cast<double>(k));
  const double bc2 = 1.0 - pow(a.beta2_d, static_cast<double>(k));
  return AdamCoef{static_cast<float>(a.lr / bc1), static_cast<float>(1.0 / sqrt(bc2)), 1.f - a.lr * a.weight_decay};
}

// One AdamW element (torch.optim.AdamW, foreach=False order): theta *= 1 - lr*wd;
// m, v EMAs of g; theta -= (lr / bc1) * m / (sqrt(v) / sqrt(bc2) + eps). Returns the change.
__device__ __forceinline__ float adamw1(const OptimArgs& a, const AdamCoef& c, float g, float& m, float& v,
                                        float& th) {
  const float old = th;
  th *= c.decay;
  m = a.beta1 * m + a.one_minus_beta1 * g;
  v = a.beta2 * v + a.one_minus_beta2 * g * g;
  th -= c.step_size * m / (sqrtf(v) * c.rsqrt_bc2 + a.eps);
  return th - old;
}

__device__ __forceinline__ float4 adamw4(const OptimArgs& a, const AdamCoef& c, long long e, const float4 G,
                                         float4& th) {
  float4 m = *reinterpret_cast<const float4*>(a.adam_m + e);
  float4 v = *reinterpret_cast<const float4*>(a.adam_v + e);
  float4 d;
  d.x = adamw1(a, c, a.scale * G.x, m.x, v.x, th.x);
  d.y = adamw1(a, c, a.scale * G.y, m.y, v.y, th.y);
  d.z = adamw1(a, c, a.scale * G.z, m.z, v.z, th.z);
  d.w = adamw1(a, c, a.scale * G.w, m.w, v.w, th.w);
  *reinterpret_cast<float4*>(a.adam_m + e) = m;
  *reinterpret_cast<float4*>(a.adam_v + e) = v;
  return d;
}

__global__ void __launch_bounds__(kBlock) masked_sgd_units_kernel(const OptimArgs a) {
  pdl_begin();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ int red[kBlock / 32];
  const bool apf = a.apf_ema != nullptr;
  for (int u = blockIdx.x; u < a.total_units; u += gridDim.x) {
    const bool touched = a.unit_stamp[u] == a.stamp;
    if (!touched && !apf) continue;  // frozen in every microbatch: no update (sandbox.cpp:250)
    AdamCoef ac{};
    if (a.adamw && touched) ac = adam_coef(a, a.unit_steps[u] + 1);
    const UnitMatrix& m = find_matrix(a.mats, a.nmats, u);
    const int lu = u - m.unit_offset;
    const int rb = lu / m.tiles_n, cb = lu - rb * m.tiles_n;
    const int r0 = rb * 128, c0 = cb * 128;
    const int nrows = min(128, m.rows - r0), ncols = min(128, m.cols - c0);
    int eligible = 0;
    const int col = lane * 4;
    if (col < ncols) {
#pragma unroll 4
      for (int r = warp; r < nrows; r += kBlock / 32) {
        const long long e = m.elem_offset + static_cast<long long>(r0 + r) * m.cols + c0 + col;
        float4 d = make_float4(0.f, 0.f, 0.f, 0.f);
        if (touched) {
          const float4 g = __ldcs(reinterpret_cast<const float4*>(a.grad + e));
          float4 th = *reinterpret_cast<const float4*>(a.master + e);
          if (a.adamw) {
            d = adamw4(a, ac, e, g, th);
          } else {
            d = make_float4(-a.scale * g.x, -a.scale * g.y, -a.scale * g.z, -a.scale * g.w);
            th.x += d.x;
            th.y += d.y;
            th.z += d.z;
            th.w += d.w;
          }
          *reinterpret_cast<float4*>(a.master + e) = th;
          uint2 packed;
          packed.x = pack_bf16x2(th.x, th.y);
          packed.y = pack_bf16x2(th.z, th.w);
          *reinterpret_cast<uint2*>(a.weights + e) = packed;
        }
        if (apf) {
          const long long i = e - a.apf_elem_base;
          float4 E = *reinterpret_cast<const float4*>(a.apf_ema + i);
          float4 A = *reinterpret_cast<const float4*>(a.apf_ema_abs + i);
          const float al = a.apf_alpha, be = 1.0f - a.apf_alpha;
          E.x = al * E.x + be * d.x;
          E.y = al * E.y + be * d.y;
          E.z = al * E.z + be * d.z;
          E.w = al * E.w + be * d.w;
          A.x = al * A.x + be * fabsf(d.x);
          A.y = al * A.y + be * fabsf(d.y);
          A.z = al * A.z + be * fabsf(d.z);
          A.w = al * A.w + be * fabsf(d.w);
          *reinterpret_cast<float4*>(a.apf_ema + i) = E;
          *reinterpret_cast<float4*>(a.apf_ema_abs + i) = A;
          auto below = [&](float ev, float av) { return (av == 0.f ? 1.f : fabsf(ev) / av) < a.apf_threshold; };
          eligible += below(E.x, A.x) + below(E.y, A.y) + below(E.z, A.z) + below(E.w, A.w);
        }
      }
    }
    if (a.adamw && touched) {  // every thread has read the old count (adam_coef) before this write
      __syncthreads();
      if (threadIdx.x == 0) a.unit_steps[u] += 1;
    }
    if (apf && a.apf_eligible != nullptr) {
      eligible = warp_isum(eligible);
      if (lane == 0) red[warp] = eligible;
      __syncthreads();
      if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < kBlock / 32; ++w) t += red[w];
        a.apf_eligible[u] = t;
      }
      __syncthreads();
    }
  }
}

__global__ void sgd_dense_kernel(float* __restrict__ master, __nv_bfloat16* __restrict__ w,
                                 const float* __restrict__ g, long long n4, float scale) {
  pdl_begin();
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const float4 gv = reinterpret_cast<const float4*>(g)[i];
    float4 t = reinterpret_cast<float4*>(master)[i];
    t.x -= scale * gv.x;
    t.y -= scale * gv.y;
    t.z -= scale * gv.z;
    t.w -= scale * gv.w;
    reinterpret_cast<float4*>(master)[i] = t;
    uint2 p;
    p.x = pack_bf16x2(t.x, t.y);
    p.y = pack_bf16x2(t.z, t.w);
    reinterpret_cast<uint2*>(w)[i] = p;
  }
}

__global__ void apf_update_kernel(float* __restrict__ ema, float* __restrict__ ema_abs,
                                  const float* __restrict__ delta, float* __restrict__ score, long long n,
                                  float alpha) {
  pdl_begin();
  const float be = 1.0f - alpha;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const float d = delta[i];
    const float e = alpha * ema[i] + be * d;
    const float a = alpha * ema_abs[i] + be * fabsf(d);
    ema[i] = e;
    ema_abs[i] = a;
    if (score) score[i] = a == 0.f ? 1.f : fabsf(e) / a;
  }
}

// ------------------------------------------------------------------ K7 glue
__global__ void embedding_fwd_kernel(const int* __restrict__ tok, const __nv_bfloat16* __restrict__ table,
                                     __nv_bfloat16* __restrict__ out, int T, int h) {
  pdl_begin();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int t = warp; t < T; t += nw) {
    const uint4* src = reinterpret_cast<const uint4*>(table + static_cast<long long>(tok[t]) * h);
    uint4* dst = reinterpret_cast<uint4*>(out + static_cast<long long>(t) * h);
    for (int c = lane; c < h / 8; c += 32) dst[c] = src[c];
  }
}

__global__ void embedding_bwd_kernel(const int* __restrict__ tok, const __nv_bfloat16* __restrict__ dout,
                                     float* __restrict__ gtable, int T, int h) {
  pdl_begin();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int t = warp; t < T; t += nw) {
    float* dst = gtable + static_cast<long long>(tok[t]) * h;
    const __nv_bfloat16* src = dout + static_cast<long long>(t) * h;
    for (int c = lane * 8; c < h; c += 256) {
      float f[8];
      load8(src + c, f);
      atomicAdd(reinterpret_cast<float4*>(dst + c), make_float4(f[0], f[1], f[2], f[3]));
      atomicAdd(reinterpret_cast<float4*>(dst + c + 4), make_float4(f[4], f[5], f[6], f[7]));
    }
  }
}

__global__ void rmsnorm_fwd_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ g,
                                   __nv_bfloat16* __restrict__ y, float* __restrict__ rstd, int T, int h,
                                   float eps) {
  pdl_begin();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int t = warp; t < T; t += nw) {
    const __nv_bfloat16* xr = x + static_cast<long long>(t) * h;
    float ss = 0.f;
    for (int c = lane * 8; c < h; c += 256) {
      float f[8];
      load8(xr + c, f);
#pragma unroll
      for (int i = 0; i < 8; ++i) ss += f[i] * f[i];
    }
    ss = warp_sum(ss);
    const float r = rsqrtf(ss / h + eps);
    if (lane == 0) rstd[t] = r;
    __nv_bfloat16* yr = y + static_cast<long long>(t) * h;
    for (int c = lane * 8; c < h; c += 256) {
      float f[8], gg[8];
      load8(xr + c, f);
      load8(g + c, gg);
#pragma unroll
      for (int i = 0; i < 8; ++i) f[i] = f[i] * r * gg[i];
      store8(yr + c, f);
    }
  }
}

// dg[c] += sum_t dy[t,c] * x[t,c] * rstd[t]: column reduction. Block = 32 column
// groups of 8 (256 columns) x 8 row lanes; each thread sums its rows in registers.
__global__ void __launch_bounds__(kBlock) rmsnorm_dg_kernel(const __nv_bfloat16* __restrict__ x,
                                                            const float* __restrict__ rstd,
                                                            const __nv_bfloat16* __restrict__ dy,
                                                            float* __restrict__ dg, int T, int h, int rows_per_block) {
  pdl_begin();
  __shared__ float part[8][256 + 4];
  const int cg = threadIdx.x & 31, rl = threadIdx.x >> 5;
  const int c = blockIdx.x * 256 + cg * 8;
  const int r0 = blockIdx.y * rows_per_block;
  const int r1 = min(T, r0 + rows_per_block);
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (c < h) {
    for (int t = r0 + rl; t < r1; t += 8) {
      float xv[8], dv[8];
      const long long off = static_cast<long long>(t) * h + c;
      load8(x + off, xv);
      load8(dy + off, dv);
      const float r = rstd[t];
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] += dv[i] * xv[i] * r;
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) part[rl][cg * 8 + i] = acc[i];
  __syncthreads();
  const int col = blockIdx.x * 256 + threadIdx.x;
  if (col < h) {
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += part[k][threadIdx.x];
    atomicAdd(&dg[col], s);
  }
}

// dx = residual + rstd * g * dy - rstd^3 * x * mean(g * dy * x); one warp per row
__global__ void __launch_bounds__(kBlock) rmsnorm_bwd_kernel(const __nv_bfloat16* __restrict__ x,
                                                             const __nv_bfloat16* __restrict__ g,
                                                             const float* __restrict__ rstd,
                                                             const __nv_bfloat16* __restrict__ dy,
                                                             const __nv_bfloat16* __restrict__ residual,
                                                             __nv_bfloat16* __restrict__ dx, int T, int h) {
  pdl_begin();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int t = blockIdx.x * (kBlock / 32) + warp; t < T; t += gridDim.x * (kBlock / 32)) {
    const long long off = static_cast<long long>(t) * h;
    const float r = rstd[t];
    float dot = 0.f;
    for (int c = lane * 8; c < h; c += 256) {
      float xv[8], gv[8], dv[8];
      load8(x + off + c, xv);
      load8(g + c, gv);
      load8(dy + off + c, dv);
#pragma unroll
      for (int i = 0; i < 8; ++i) dot += gv[i] * dv[i] * xv[i];
    }
    dot = warp_sum(dot);
    const float k = dot * r * r * r / h;
    for (int c = lane * 8; c < h; c += 256) {
      float xv[8], gv[8], dv[8], out[8];
      load8(x + off + c, xv);
      load8(g + c, gv);
      load8(dy + off + c, dv);
      if (residual) load8(residual + off + c, out);
#pragma unroll
      for (int i = 0; i < 8; ++i) out[i] = (residual ? out[i] : 0.f) + r * gv[i] * dv[i] - k * xv[i];
      store8(dx + off + c, out);
    }
  }
}

// Row-in-registers RMSNorm for h = 256 * CH (the LLaMA widths): one warp per row, lane
// holds columns lane*8 + 256 j (16-byte loads), so x is read from HBM exactly once.
template <int CH>
__global__ void __launch_bounds__(kBlock) rmsnorm_fwd_reg_kernel(const __nv_bfloat16* __restrict__ x,
                                                                 const __nv_bfloat16* __restrict__ g,
                                                                 __nv_bfloat16* __restrict__ y,
                                                                 float* __restrict__ rstd, int T, float eps) {
  pdl_begin();
  constexpr int H = 256 * CH;
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < T; t += nw) {
    const __nv_bfloat16* xr = x + static_cast<long long>(t) * H + lane * 8;
    uint4 xv[CH], gv[CH];  // g rides with x: its loads do not wait behind the row reduction
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      xv[j] = __ldcs(reinterpret_cast<const uint4*>(xr + 256 * j));
      gv[j] = *reinterpret_cast<const uint4*>(g + lane * 8 + 256 * j);
    }
    float ss = 0.f;
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&xv[j]);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(b[i]);
        ss += f.x * f.x + f.y * f.y;
      }
    }
    ss = warp_sum(ss);
    const float r = rsqrtf(ss / H + eps);
    if (lane == 0) rstd[t] = r;
    __nv_bfloat16* yr = y + static_cast<long long>(t) * H + lane * 8;
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      float f[8], gg[8];
      const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&xv[j]);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 v = __bfloat1622float2(b[i]);
        f[2 * i] = v.x;
        f[2 * i + 1] = v.y;
      }
      const __nv_bfloat162* gb = reinterpret_cast<const __nv_bfloat162*>(&gv[j]);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 v = __bfloat1622float2(gb[i]);
        gg[2 * i] = v.x;
        gg[2 * i + 1] = v.y;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) f[i] = f[i] * r * gg[i];
      store8(yr + 256 * j, f);
    }
  }
}

// Fused RMSNorm backward for h = 256 * CH: dx = residual + rstd * g * dy - rstd^3 * x * mean(g * dy * x)
// and dg[c] += sum_t dy[t,c] * x[t,c] * rstd[t] in ONE pass over x and dy (was two kernels).
// One warp per row; rows are held in registers (CH <= 8). A warp's dg partial lives in
// registers (CH <= 4) or in its shared-memory slice; the block's slices are summed and
// added to dg with one float4 atomic per 4 columns (148 blocks: ~77k vector atomics).
template <int CH>
__host__ __device__ constexpr int norm_bwd_threads() { return 256; }

template <int CH>
__global__ void __launch_bounds__(norm_bwd_threads<CH>(), 1) rmsnorm_bwd_fused_kernel(
    const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ g, const float* __restrict__ rstd,
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ residual, __nv_bfloat16* __restrict__ dx,
    float* __restrict__ dg, int T) {
  pdl_begin();
  constexpr int H = 256 * CH;
  constexpr int NT = norm_bwd_threads<CH>();
  constexpr int NW = NT / 32;
  constexpr bool ACC_REG = CH <= 4;  // dg partial in registers (else in the warp's smem slice)
  constexpr bool HOLD = CH <= 8;     // x and dy kept in registers between the two passes (else re-read)
  extern __shared__ float slices[];  // [NW][H]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* mine = slices + warp * H + lane * 8;
  float acc[ACC_REG ? CH * 8 : 1];
  if constexpr (ACC_REG) {
#pragma unroll
    for (int i = 0; i < CH * 8; ++i) acc[i] = 0.f;
  } else {
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      reinterpret_cast<float4*>(mine + 256 * j)[0] = make_float4(0.f, 0.f, 0.f, 0.f);
      reinterpret_cast<float4*>(mine + 256 * j)[1] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  for (int t = blockIdx.x * NW + warp; t < T; t += gridDim.x * NW) {
    const long long off = static_cast<long long>(t) * H + lane * 8;
    uint4 xv[HOLD ? CH : 1], dv[HOLD ? CH : 1], rv[HOLD ? CH : 1];
    if constexpr (HOLD) {  // the residual rides with x: one memory round trip per row
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        xv[j] = __ldcs(reinterpret_cast<const uint4*>(x + off + 256 * j));
        if (residual) rv[j] = __ldcs(reinterpret_cast<const uint4*>(residual + off + 256 * j));
      }
    }
    const float r = rstd[t];
    float dot = 0.f;
#pragma unroll(HOLD ? CH : 4)
    for (int j = 0; j < CH; ++j) {
      float gv[8];
      load8(g + lane * 8 + 256 * j, gv);
      uint4 xj;
      if constexpr (HOLD) xj = xv[j];
      else xj = *reinterpret_cast<const uint4*>(x + off + 256 * j);
      const uint4 dj = *reinterpret_cast<const uint4*>(dy + off + 256 * j);
      if constexpr (HOLD) dv[j] = dj;
      const __nv_bfloat162* xb = reinterpret_cast<const __nv_bfloat162*>(&xj);
      const __nv_bfloat162* db = reinterpret_cast<const __nv_bfloat162*>(&dj);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 xf = __bfloat1622float2(xb[i]), df = __bfloat1622float2(db[i]);
        dot += gv[2 * i] * df.x * xf.x + gv[2 * i + 1] * df.y * xf.y;
      }
    }
    dot = warp_sum(dot);
    const float k = dot * r * r * r / H;
#pragma unroll(HOLD ? CH : 4)
    for (int j = 0; j < CH; ++j) {
      float gv[8], out[8];
      load8(g + lane * 8 + 256 * j, gv);
      if (residual) {
        if constexpr (HOLD) {
          const __nv_bfloat162* r2 = reinterpret_cast<const __nv_bfloat162*>(&rv[j]);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float2 t2 = __bfloat1622float2(r2[i]);
            out[2 * i] = t2.x;
            out[2 * i + 1] = t2.y;
          }
        } else {
          load8(residual + off + 256 * j, out);
        }
      }
      uint4 xj, dj;
      if constexpr (HOLD) {
        xj = xv[j];
        dj = dv[j];
      } else {
        xj = __ldcs(reinterpret_cast<const uint4*>(x + off + 256 * j));
        dj = __ldcs(reinterpret_cast<const uint4*>(dy + off + 256 * j));
      }
      const __nv_bfloat162* xb = reinterpret_cast<const __nv_bfloat162*>(&xj);
      const __nv_bfloat162* db = reinterpret_cast<const __nv_bfloat162*>(&dj);
      float c[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 xf = __bfloat1622float2(xb[i]), df = __bfloat1622float2(db[i]);
        out[2 * i] = (residual ? out[2 * i] : 0.f) + r * gv[2 * i] * df.x - k * xf.x;
        out[2 * i + 1] = (residual ? out[2 * i + 1] : 0.f) + r * gv[2 * i + 1] * df.y - k * xf.y;
        c[2 * i] = df.x * xf.x * r;
        c[2 * i + 1] = df.y * xf.y * r;
      }
      store8(dx + off + 256 * j, out);
      if constexpr (ACC_REG) {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[8 * j + i] += c[i];
      } else {
        float4* m4 = reinterpret_cast<float4*>(mine + 256 * j);
        const float4 a = m4[0], b = m4[1];
        m4[0] = make_float4(a.x + c[0], a.y + c[1], a.z + c[2], a.w + c[3]);
        m4[1] = make_float4(b.x + c[4], b.y + c[5], b.z + c[6], b.w + c[7]);
      }
    }
  }
  if (dg == nullptr) return;
  if constexpr (ACC_REG) {
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      reinterpret_cast<float4*>(mine + 256 * j)[0] = make_float4(acc[8 * j], acc[8 * j + 1], acc[8 * j + 2], acc[8 * j + 3]);
      reinterpret_cast<float4*>(mine + 256 * j)[1] =
          make_float4(acc[8 * j + 4], acc[8 * j + 5], acc[8 * j + 6], acc[8 * j + 7]);
    }
  }
  __syncthreads();
  // block partial (slices summed in warp order) -> dg with one vector atomic per 4 columns
  for (int c = threadIdx.x * 4; c < H; c += NT * 4) {
    float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const float4 v = *reinterpret_cast<const float4*>(slices + w * H + c);
      sum = make_float4(sum.x + v.x, sum.y + v.y, sum.z + v.z, sum.w + v.w);
    }
    atomicAdd(reinterpret_cast<float4*>(dg + c), sum);
  }
}

// RMSNorm for the LLaMA-8B / 13B hidden sizes (h = 256 CH, CH = 16, 20): one thread per 8 columns of
// a row (a block of CH warps spans the row), R rows per iteration. Every load of an iteration is issued
// before the row reductions (R rows x {x, dy, residual} x 16 B per thread in flight); the per-row sums
// are combined across the block's warps through a double-buffered shared array with ONE barrier per
// R rows. The backward's dg partial stays in the thread's 8 registers for all of the block's rows and
// leaves with two float4 atomics per thread. The warp-per-row kernels above re-read x / dy from L1/L2
// in a second pass and kept dg in shared memory at these sizes (2.5x their HBM time, 8B step ncu).
template <int CH, int R>
__global__ void __launch_bounds__(CH * 32) rmsnorm_fwd_rows_kernel(const __nv_bfloat16* __restrict__ x,
                                                                   const __nv_bfloat16* __restrict__ g,
                                                                   __nv_bfloat16* __restrict__ y,
                                                                   float* __restrict__ rstd, int T, float eps) {
  pdl_begin();
  constexpr int H = 256 * CH;
  __shared__ float red[2][R][CH];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int col = threadIdx.x * 8;
  float gv[8];
  load8(g + col, gv);
  int buf = 0;
  for (int t0 = blockIdx.x * R; t0 < T; t0 += gridDim.x * R, buf ^= 1) {
    uint4 xv[R];
#pragma unroll
    for (int q = 0; q < R; ++q)
      xv[q] = t0 + q < T ? __ldcs(reinterpret_cast<const uint4*>(x + static_cast<long long>(t0 + q) * H + col))
                         : make_uint4(0u, 0u, 0u, 0u);
    float ss[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&xv[q]);
      float a = 0.f;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(b[i]);
        a += f.x * f.x + f.y * f.y;
      }
      ss[q] = warp_sum(a);
    }
    if (lane == 0) {
#pragma unroll
      for (int q = 0; q < R; ++q) red[buf][q][warp] = ss[q];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int t = t0 + q;
      if (t >= T) break;
      float tot = 0.f;
#pragma unroll
      for (int w = 0; w < CH; ++w) tot += red[buf][q][w];
      const float r = rsqrtf(tot / H + eps);
      if (threadIdx.x == 0) rstd[t] = r;
      const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&xv[q]);
      float f[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 v = __bfloat1622float2(b[i]);
        f[2 * i] = v.x * r * gv[2 * i];
        f[2 * i + 1] = v.y * r * gv[2 * i + 1];
      }
      store8(y + static_cast<long long>(t) * H + col, f);
    }
  }
}

template <int CH, int R>
__global__ void __launch_bounds__(CH * 32) rmsnorm_bwd_rows_kernel(
    const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ g, const float* __restrict__ rstd,
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ residual, __nv_bfloat16* __restrict__ dx,
    float* __restrict__ dg, int T) {
  pdl_begin();
  constexpr int H = 256 * CH;
  __shared__ float red[2][R][CH];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int col = threadIdx.x * 8;
  float gv[8], acc[8];
  load8(g + col, gv);
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.f;
  int buf = 0;
  for (int t0 = blockIdx.x * R; t0 < T; t0 += gridDim.x * R, buf ^= 1) {
    uint4 xv[R], dv[R], rv[R];
    float rr[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const bool ok = t0 + q < T;
      const long long off = static_cast<long long>(t0 + q) * H + col;
      const uint4 z = make_uint4(0u, 0u, 0u, 0u);
      xv[q] = ok ? __ldcs(reinterpret_cast<const uint4*>(x + off)) : z;
      dv[q] = ok ? __ldcs(reinterpret_cast<const uint4*>(dy + off)) : z;
      rv[q] = ok && residual ? __ldcs(reinterpret_cast<const uint4*>(residual + off)) : z;
      rr[q] = ok ? rstd[t0 + q] : 0.f;
    }
    float dot[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const __nv_bfloat162* xb = reinterpret_cast<const __nv_bfloat162*>(&xv[q]);
      const __nv_bfloat162* db = reinterpret_cast<const __nv_bfloat162*>(&dv[q]);
      float a = 0.f;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 xf = __bfloat1622float2(xb[i]), df = __bfloat1622float2(db[i]);
        a += gv[2 * i] * df.x * xf.x + gv[2 * i + 1] * df.y * xf.y;
      }
      dot[q] = warp_sum(a);
    }
    if (lane == 0) {
#pragma unroll
      for (int q = 0; q < R; ++q) red[buf][q][warp] = dot[q];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int t = t0 + q;
      if (t >= T) break;
      float tot = 0.f;
#pragma unroll
      for (int w = 0; w < CH; ++w) tot += red[buf][q][w];
      const float r = rr[q];
      const float k = tot * r * r * r / H;
      const __nv_bfloat162* xb = reinterpret_cast<const __nv_bfloat162*>(&xv[q]);
      const __nv_bfloat162* db = reinterpret_cast<const __nv_bfloat162*>(&dv[q]);
      const __nv_bfloat162* rb = reinterpret_cast<const __nv_bfloat162*>(&rv[q]);
      float out[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 xf = __bfloat1622float2(xb[i]), df = __bfloat1622float2(db[i]);
        const float2 rf = __bfloat1622float2(rb[i]);
        out[2 * i] = rf.x + r * gv[2 * i] * df.x - k * xf.x;
        out[2 * i + 1] = rf.y + r * gv[2 * i + 1] * df.y - k * xf.y;
        acc[2 * i] += df.x * xf.x * r;
        acc[2 * i + 1] += df.y * xf.y * r;
      }
      store8(dx + static_cast<long long>(t) * H + col, out);
    }
  }
  if (dg == nullptr) return;
  atomicAdd(reinterpret_cast<float4*>(dg + col), make_float4(acc[0], acc[1], acc[2], acc[3]));
  atomicAdd(reinterpret_cast<float4*>(dg + col + 4), make_float4(acc[4], acc[5], acc[6], acc[7]));
}

// Software-pipelined RMSNorm forward at h = 256 CH: the next batch of R rows is loaded under the
// current batch's reduction and stores.
template <int CH, int R>
__global__ void __launch_bounds__(CH * 32) rmsnorm_fwd_pipe_kernel(const __nv_bfloat16* __restrict__ x,
                                                                   const __nv_bfloat16* __restrict__ g,
                                                                   __nv_bfloat16* __restrict__ y,
                                                                   float* __restrict__ rstd, int T, float eps) {
  pdl_begin();
  constexpr int H = 256 * CH;
  __shared__ float red[2][R][CH];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int col = threadIdx.x * 8;
  float gv[8];
  load8(g + col, gv);
  uint4 xv[R];
  auto fetch = [&](int t0) {
#pragma unroll
    for (int q = 0; q < R; ++q)
      xv[q] = t0 + q < T ? __ldcs(reinterpret_cast<const uint4*>(x + static_cast<long long>(t0 + q) * H + col))
                         : make_uint4(0u, 0u, 0u, 0u);
  };
  int buf = 0;
  int t0 = blockIdx.x * R;
  if (t0 < T) fetch(t0);
  for (; t0 < T; t0 += gridDim.x * R, buf ^= 1) {
    uint4 cx[R];
#pragma unroll
    for (int q = 0; q < R; ++q) cx[q] = xv[q];
    const int tn = t0 + gridDim.x * R;
    if (tn < T) fetch(tn);
    float ss[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&cx[q]);
      float a = 0.f;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(b[i]);
        a += f.x * f.x + f.y * f.y;
      }
      ss[q] = warp_sum(a);
    }
    if (lane == 0) {
#pragma unroll
      for (int q = 0; q < R; ++q) red[buf][q][warp] = ss[q];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int t = t0 + q;
      if (t >= T) break;
      float tot = 0.f;
#pragma unroll
      for (int w = 0; w < CH; ++w) tot += red[buf][q][w];
      const float r = rsqrtf(tot / H + eps);
      if (threadIdx.x == 0) rstd[t] = r;
      const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&cx[q]);
      float f[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 v = __bfloat1622float2(b[i]);
        f[2 * i] = v.x * r * gv[2 * i];
        f[2 * i + 1] = v.y * r * gv[2 * i + 1];
      }
      store8(y + static_cast<long long>(t) * H + col, f);
    }
  }
}

// Software-pipelined RMSNorm backward at h = 256 CH: the loads of the CTA's next R rows are issued
// before the current rows' reductions, barrier and stores, so a CTA always has a batch of rows in
// flight (the row-block kernel above waits for each batch's loads).
template <int CH, int R>
__global__ void __launch_bounds__(CH * 32) rmsnorm_bwd_pipe_kernel(
    const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ g, const float* __restrict__ rstd,
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ residual, __nv_bfloat16* __restrict__ dx,
    float* __restrict__ dg, int T) {
  pdl_begin();
  constexpr int H = 256 * CH;
  __shared__ float red[2][R][CH];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int col = threadIdx.x * 8;
  float gv[8], acc[8];
  load8(g + col, gv);
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.f;
  const uint4 z = make_uint4(0u, 0u, 0u, 0u);
  uint4 xv[R], dv[R], rv[R];
  float rr[R];
  auto fetch = [&](int t0) {
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const bool ok = t0 + q < T;
      const long long off = static_cast<long long>(t0 + q) * H + col;
      xv[q] = ok ? __ldcs(reinterpret_cast<const uint4*>(x + off)) : z;
      dv[q] = ok ? __ldcs(reinterpret_cast<const uint4*>(dy + off)) : z;
      rv[q] = ok && residual ? __ldcs(reinterpret_cast<const uint4*>(residual + off)) : z;
      rr[q] = ok ? rstd[t0 + q] : 0.f;
    }
  };
  int buf = 0;
  int t0 = blockIdx.x * R;
  if (t0 < T) fetch(t0);
  for (; t0 < T; t0 += gridDim.x * R, buf ^= 1) {
    uint4 cx[R], cd[R], cres[R];
    float cr[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      cx[q] = xv[q];
      cd[q] = dv[q];
      cres[q] = rv[q];
      cr[q] = rr[q];
    }
    const int tn = t0 + gridDim.x * R;
    if (tn < T) fetch(tn);  // next batch in flight under this one
    float dot[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const __nv_bfloat162* xb = reinterpret_cast<const __nv_bfloat162*>(&cx[q]);
      const __nv_bfloat162* db = reinterpret_cast<const __nv_bfloat162*>(&cd[q]);
      float a = 0.f;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 xf = __bfloat1622float2(xb[i]), df = __bfloat1622float2(db[i]);
        a += gv[2 * i] * df.x * xf.x + gv[2 * i + 1] * df.y * xf.y;
      }
      dot[q] = warp_sum(a);
    }
    if (lane == 0) {
#pragma unroll
      for (int q = 0; q < R; ++q) red[buf][q][warp] = dot[q];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int t = t0 + q;
      if (t >= T) break;
      float tot = 0.f;
#pragma unroll
      for (int w = 0; w < CH; ++w) tot += red[buf][q][w];
      const float r = cr[q];
      const float k = tot * r * r * r / H;
      const __nv_bfloat162* xb = reinterpret_cast<const __nv_bfloat162*>(&cx[q]);
      const __nv_bfloat162* db = reinterpret_cast<const __nv_bfloat162*>(&cd[q]);
      const __nv_bfloat162* rb = reinterpret_cast<const __nv_bfloat162*>(&cres[q]);
      float out[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 xf = __bfloat1622float2(xb[i]), df = __bfloat1622float2(db[i]);
        const float2 rf = __bfloat1622float2(rb[i]);
        out[2 * i] = rf.x + r * gv[2 * i] * df.x - k * xf.x;
        out[2 * i + 1] = rf.y + r * gv[2 * i + 1] * df.y - k * xf.y;
        acc[2 * i] += df.x * xf.x * r;
        acc[2 * i + 1] += df.y * xf.y * r;
      }
      store8(dx + static_cast<long long>(t) * H + col, out);
    }
  }
  if (dg == nullptr) return;
  atomicAdd(reinterpret_cast<float4*>(dg + col), make_float4(acc[0], acc[1], acc[2], acc[3]));
  atomicAdd(reinterpret_cast<float4*>(dg + col + 4), make_float4(acc[4], acc[5], acc[6], acc[7]));
}

// rotate-half RoPE on the q and k heads of the packed qkv activation, in place.
// grid.y = token; each thread rotates 8 consecutive pairs (16-byte loads).
__global__ void rope_fwd_kernel(__nv_bfloat16* __restrict__ qkv, const float2* __restrict__ cs, int seq, int nh,
                                int nkv, int hd) {
  pdl_begin();
  const int half = hd / 2, chunks = half / 8;
  const int t = blockIdx.y;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (nh + nkv) * chunks) return;
  const int head = idx / chunks, j = (idx - head * chunks) * 8;
  __nv_bfloat16* p = qkv + static_cast<long long>(t) * (nh + 2 * nkv) * hd + static_cast<long long>(head) * hd;
  const float2* c = cs + static_cast<long long>(t % seq) * half + j;
  float a[8], b[8], oa[8], ob[8];
  load8(p + j, a);
  load8(p + j + half, b);
#pragma unroll
  for (int i = 0; i < 8; ++i) rope_rotate(a[i], b[i], c[i], oa[i], ob[i]);
  store8(p + j, oa);
  store8(p + j + half, ob);
}

__device__ __forceinline__ float sigmoidf_(float x) { return sigmoid_fast(x); }

// gate|up rows are interleaved in 128-blocks (kGuBlock): gu column of gate j is
// (j / 128) * 256 + j % 128, up j sits 128 further (so one 256-wide GEMM tile holds
// matching gate and up columns and the GEMM epilogue can apply SwiGLU).
__device__ __forceinline__ int gate_col(int j) { return ((j >> 7) << 8) + (j & 127); }

// grid.y = token, x covers the row in 8-element chunks (no 64-bit index division)
__global__ void swiglu_fwd_kernel(const __nv_bfloat16* __restrict__ gu, __nv_bfloat16* __restrict__ a, int T,
                                  int ffn) {
  pdl_begin();
  {
    const long long t = blockIdx.y;
    const int c = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
    if (c >= ffn) return;
    float g[8], u[8], o[8];
    const __nv_bfloat16* row = gu + t * 2 * ffn + gate_col(c);
    load8(row, g);
    load8(row + 128, u);
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] = g[k] * sigmoidf_(g[k]) * u[k];
    store8(a + t * ffn + c, o);
  }
}

__global__ void swiglu_bwd_kernel(const __nv_bfloat16* __restrict__ gu, const __nv_bfloat16* __restrict__ da,
                                  __nv_bfloat16* __restrict__ dgu, int T, int ffn) {
  pdl_begin();
  {
    const long long t = blockIdx.y;
    const int c = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
    if (c >= ffn) return;
    float g[8], u[8], d[8], dg[8], du[8];
    const long long off = t * 2 * ffn + gate_col(c);
    load8(gu + off, g);
    load8(gu + off + 128, u);
    load8(da + t * ffn + c, d);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float s = sigmoidf_(g[k]);
      const float silu = g[k] * s;
      du[k] = d[k] * silu;
      dg[k] = d[k] * u[k] * s * (1.f + g[k] * (1.f - s));
    }
    store8(dgu + off, dg);
    store8(dgu + off + 128, du);
  }
}

// One block per row: online max/sum-exp, then dlogits in place. Large vocabularies use
// 512-thread blocks, 2 per SM: ~300 rows in flight (76 MB at V = 128256) stay in L2, so the
// second pass over a row hits L2 instead of HBM (with 8 x 256-thread blocks per SM, 1184 rows
// = 303 MB were in flight and the row was read from HBM twice). Four 16-byte loads per
// thread are issued before their max/exp work.
constexpr float kLog2e = 1.4426950408889634f;
__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

template <int NT>
__global__ void __launch_bounds__(NT, NT >= 512 ? 2 : 1) cross_entropy_kernel(__nv_bfloat16* __restrict__ logits,
                                                                             const int* __restrict__ targets,
                                                                             float* __restrict__ loss_sum, int V,
                                                                             float grad_scale, float loss_scale) {
  pdl_begin();
  const long long t = blockIdx.x;
  __nv_bfloat16* row = logits + t * V;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ float sm[NT / 32], ss[NT / 32];
  float mx = -INFINITY, sum = 0.f;
  constexpr int U = 4;
  for (int c0 = threadIdx.x * 8; c0 < V; c0 += NT * 8 * U) {
    uint4 raw[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = c0 + u * NT * 8;
      raw[u] = c < V ? *reinterpret_cast<const uint4*>(row + c)
                     : make_uint4(0xff80ff80u, 0xff80ff80u, 0xff80ff80u, 0xff80ff80u);  // bf16 -inf
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float f[8];
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw[u]);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 v2 = __bfloat1622float2(h[i]);
        f[2 * i] = v2.x;
        f[2 * i + 1] = v2.y;
      }
      float lm = f[0];
#pragma unroll
      for (int i = 1; i < 8; ++i) lm = fmaxf(lm, f[i]);
      if (lm == -INFINITY) continue;  // padding chunk past the row end
      const float nm = fmaxf(mx, lm);
      // e^(x - m) = 2^(x log2e - m log2e): one FFMA + one MUFU.EX2 per logit
      const float nml = nm * kLog2e;
      sum *= ex2_approx(fmaf(mx, kLog2e, -nml));
#pragma unroll
      for (int i = 0; i < 8; ++i) sum += ex2_approx(fmaf(f[i], kLog2e, -nml));
      mx = nm;
    }
  }
  // combine (max, sum) across the block
  float wm = warp_max(mx);
  // threads (or whole warps) without elements carry mx = -inf, sum = 0
  float ws = warp_sum(mx == -INFINITY ? 0.f : sum * __expf(mx - wm));
  if (lane == 0) {
    sm[warp] = wm;
    ss[warp] = ws;
  }
  __syncthreads();
  float bm = -INFINITY;
  for (int w = 0; w < NT / 32; ++w) bm = fmaxf(bm, sm[w]);
  float bs = 0.f;
  for (int w = 0; w < NT / 32; ++w) bs += sm[w] == -INFINITY ? 0.f : ss[w] * __expf(sm[w] - bm);
  const float lse = bm + __logf(bs);
  const int tgt = targets[t];
  const float xt = __bfloat162float(row[tgt]);
  __syncthreads();
  const float lsel = lse * kLog2e;
  for (int c = threadIdx.x * 8; c < V; c += NT * 8) {
    float f[8];
    load8(row + c, f);
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = (ex2_approx(fmaf(f[i], kLog2e, -lsel)) - (c + i == tgt ? 1.f : 0.f)) * grad_scale;
    store8(row + c, f);
  }
  if (threadIdx.x == 0) atomicAdd(loss_sum, (lse - xt) * loss_scale);
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__global__ void init_normal_kernel(float* __restrict__ master, __nv_bfloat16* __restrict__ w, long long n,
                                   float stddev, uint64_t seed) {
  pdl_begin();
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const uint64_t r = mix64(seed + 0x9e3779b97f4a7c15ULL * static_cast<uint64_t>(i + 1));
    const float u1 = (static_cast<float>(r >> 40) + 1.0f) * (1.0f / 16777217.0f);
    const float u2 = static_cast<float>((r >> 16) & 0xFFFFFF) * (1.0f / 16777216.0f);
    const float v = stddev * sqrtf(-2.f * __logf(u1)) * __cosf(6.28318530718f * u2);
    master[i] = v;
    w[i] = __float2bfloat16_rn(v);
  }
}

__global__ void fill_kernel(float* __restrict__ master, __nv_bfloat16* __restrict__ w, long long n, float v) {
  pdl_begin();
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    master[i] = v;
    w[i] = __float2bfloat16_rn(v);
  }
}

__global__ void rope_table_kernel(float2* cs, int seq, int hd, float theta) {
  pdl_begin();
  const int half = hd / 2;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < seq * half; i += gridDim.x * blockDim.x) {
    const int p = i / half, j = i % half;
    const double inv = pow(static_cast<double>(theta), -2.0 * j / hd);
    const double ang = p * inv;
    cs[i] = make_float2(static_cast<float>(cos(ang)), static_cast<float>(sin(ang)));
  }
}

__global__ void random_tokens_kernel(int* tok, long long n, int vocab, uint64_t seed) {
  pdl_begin();
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    tok[i] = static_cast<int>(mix64(seed + 0x9e3779b97f4a7c15ULL * static_cast<uint64_t>(i + 1)) %
                              static_cast<uint64_t>(vocab));
}

}  // namespace

int launch_mask_to_unit_lists(const uint64_t* words, const UnitMatrix* mats, int nmats, int* lists, int* counts,
                              cudaStream_t s) {
  if (nmats <= 0) return PF_OK;
  launch_k(mask_to_lists_kernel, dim3(nmats), dim3(kBlock), 0, s, words, mats, lists, counts);
  return status();
}

int launch_mask_to_pair_lists(const uint64_t* words, const UnitMatrix* mats, int nmats, int* pairs, int* counts,
                              cudaStream_t s) {
  if (nmats <= 0) return PF_OK;
  launch_k(mask_to_pairs_kernel, dim3(nmats), dim3(kBlock), 0, s, words, mats, pairs, counts);
  return status();
}

int launch_mask_to_rowpair_lists(const uint64_t* words, const UnitMatrix* mats, int nmats, int* lists, int* counts,
                                 cudaStream_t s) {
  if (nmats <= 0) return PF_OK;
  launch_k(mask_to_rowpairs_kernel, dim3(nmats), dim3(kRowPairThreads), 0, s, words, mats, lists, counts);
  return status();
}

int launch_masked_sgd_units(const OptimArgs& a, cudaStream_t s) {
  if (a.total_units <= 0) return PF_OK;
  launch_k(masked_sgd_units_kernel, dim3(grid_for(a.total_units, 8)), dim3(kBlock), 0, s, a);
  return status();
}

int launch_sgd_dense(float* master, __nv_bfloat16* w, const float* g, long long n, float scale, cudaStream_t s) {
  if (n <= 0) return PF_OK;
  if (n % 4) return PF_ERR_INVALID;
  launch_k(sgd_dense_kernel, dim3(grid_for((n / 4 + kBlock - 1) / kBlock)), dim3(kBlock), 0, s, master, w, g, n / 4, scale);
  return status();
}

__global__ void adamw_dense_kernel(float* __restrict__ master, __nv_bfloat16* __restrict__ w,
                                   const float* __restrict__ g, float* __restrict__ m, float* __restrict__ v,
                                   long long n, const OptimArgs a, const AdamCoef c) {
  pdl_begin();
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    float th = master[i], mi = m[i], vi = v[i];
    adamw1(a, c, a.scale * g[i], mi, vi, th);
    master[i] = th;
    m[i] = mi;
    v[i] = vi;
    w[i] = __float2bfloat16_rn(th);
  }
}

int launch_adamw_dense(float* master, __nv_bfloat16* w, const float* g, float* m, float* v, long long n, float scale,
                       float lr, float beta1, float beta2, float one_minus_beta1, float one_minus_beta2, float eps,
                       float weight_decay, double bc1, double bc2, cudaStream_t s) {
  if (n <= 0) return PF_OK;
  OptimArgs a{};
  a.scale = scale;
  a.lr = lr;
  a.beta1 = beta1;
  a.beta2 = beta2;
  a.one_minus_beta1 = one_minus_beta1;
  a.one_minus_beta2 = one_minus_beta2;
  a.eps = eps;
  a.weight_decay = weight_decay;
  const AdamCoef c{static_cast<float>(lr / bc1), static_cast<float>(1.0 / std::sqrt(bc2)), 1.f - lr * weight_decay};
  launch_k(adamw_dense_kernel, dim3(grid_for((n + kBlock - 1) / kBlock)), dim3(kBlock), 0, s, master, w, g, m, v, n, a, c);
  return status();
}

int launch_apf_update(float* ema, float* ema_abs, const float* delta, float* score, long long n, float alpha,
                      cudaStream_t s) {
  if (n <= 0) return PF_OK;
  launch_k(apf_update_kernel, dim3(grid_for((n + kBlock - 1) / kBlock)), dim3(kBlock), 0, s, ema, ema_abs, delta, score, n, alpha);
  return status();
}

int launch_embedding_fwd(const int* tok, const __nv_bfloat16* table, __nv_bfloat16* out, int T, int h,
                         cudaStream_t s) {
  if (h % 8) return PF_ERR_INVALID;
  launch_k(embedding_fwd_kernel, dim3(grid_for((T + 7) / 8)), dim3(kBlock), 0, s, tok, table, out, T, h);
  return status();
}

int launch_embedding_bwd(const int* tok, const __nv_bfloat16* dout, float* g, int T, int h, cudaStream_t s) {
  if (h % 8) return PF_ERR_INVALID;
  launch_k(embedding_bwd_kernel, dim3(grid_for((T + 7) / 8)), dim3(kBlock), 0, s, tok, dout, g, T, h);
  return status();
}

// PF_NORM_ROWS=0: the warp-per-row kernels at h = 4096 too (same-process A/B in tools/norm_bench.py)
static bool norm_batch_wait() {  // PF_NORM_ROWS=1: the row-block backward without prefetch (A/B)
  const char* e = std::getenv("PF_NORM_ROWS");
  return e && e[0] == '1';
}
static bool norm_rows_off() {
  const char* e = std::getenv("PF_NORM_ROWS");
  return e && e[0] == '0';
}

int launch_rmsnorm_fwd(const __nv_bfloat16* x, const __nv_bfloat16* g, __nv_bfloat16* y, float* rstd, int T, int h,
                       float eps, cudaStream_t s) {
  if (h % 8) return PF_ERR_INVALID;
  const int grid = grid_for((T + 7) / 8);
  switch (h) {
    case 256: launch_k(rmsnorm_fwd_reg_kernel<1>, dim3(grid), dim3(kBlock), 0, s, x, g, y, rstd, T, eps); return status();
    case 512: launch_k(rmsnorm_fwd_reg_kernel<2>, dim3(grid), dim3(kBlock), 0, s, x, g, y, rstd, T, eps); return status();
    case 1024: launch_k(rmsnorm_fwd_reg_kernel<4>, dim3(grid), dim3(kBlock), 0, s, x, g, y, rstd, T, eps); return status();
    case 2048: launch_k(rmsnorm_fwd_reg_kernel<8>, dim3(grid), dim3(kBlock), 0, s, x, g, y, rstd, T, eps); return status();
    case 4096:
      if (norm_rows_off()) {
        launch_k(rmsnorm_fwd_reg_kernel<16>, dim3(grid), dim3(kBlock), 0, s, x, g, y, rstd, T, eps);
        return status();
      }
      if (!norm_batch_wait()) {
        launch_k(rmsnorm_fwd_pipe_kernel<16, 4>, dim3(std::max(1, std::min(2 * num_sms(), (T + 3) / 4))), dim3(512), 0,
                 s, x, g, y, rstd, T, eps);
        return status();
      }
      launch_k(rmsnorm_fwd_rows_kernel<16, 4>, dim3(std::max(1, std::min(2 * num_sms(), (T + 3) / 4))), dim3(512), 0, s,
               x, g, y, rstd, T, eps);
      return status();
    case 5120:
      if (!norm_batch_wait()) {
        launch_k(rmsnorm_fwd_pipe_kernel<20, 2>, dim3(std::max(1, std::min(2 * num_sms(), (T + 1) / 2))), dim3(640), 0,
                 s, x, g, y, rstd, T, eps);
        return status();
      }
      launch_k(rmsnorm_fwd_rows_kernel<20, 2>, dim3(std::max(1, std::min(2 * num_sms(), (T + 1) / 2))), dim3(640), 0, s,
               x, g, y, rstd, T, eps);
      return status();
    default: break;
  }
  launch_k(rmsnorm_fwd_kernel, dim3(grid), dim3(kBlock), 0, s, x, g, y, rstd, T, h, eps);
  return status();
}

namespace {
template <int CH>
int launch_rmsnorm_bwd_fused(const __nv_bfloat16* x, const __nv_bfloat16* g, const float* rstd,
                             const __nv_bfloat16* dy, const __nv_bfloat16* residual, __nv_bfloat16* dx, float* dg,
                             int T, cudaStream_t s) {
  constexpr int H = 256 * CH;
  constexpr int NT = norm_bwd_threads<CH>();
  constexpr int smem = (NT / 32) * H * 4;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(rmsnorm_bwd_fused_kernel<CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
        cudaSuccess)
      return PF_ERR_CUDA;
    attr = true;
  }
  const int grid = std::max(1, std::min(num_sms(), (T + NT / 32 - 1) / (NT / 32)));
  launch_k(rmsnorm_bwd_fused_kernel<CH>, dim3(grid), dim3(NT), smem, s, x, g, rstd, dy, residual, dx, dg, T);
  return status();
}
}  // namespace

int launch_rmsnorm_bwd(const __nv_bfloat16* x, const __nv_bfloat16* g, const float* rstd, const __nv_bfloat16* dy,
                       const __nv_bfloat16* residual, __nv_bfloat16* dx, float* dg, int T, int h, cudaStream_t s) {
  if (h % 8) return PF_ERR_INVALID;
  switch (h) {
    case 256: return launch_rmsnorm_bwd_fused<1>(x, g, rstd, dy, residual, dx, dg, T, s);
    case 512: return launch_rmsnorm_bwd_fused<2>(x, g, rstd, dy, residual, dx, dg, T, s);
    case 1024: return launch_rmsnorm_bwd_fused<4>(x, g, rstd, dy, residual, dx, dg, T, s);
    case 2048: return launch_rmsnorm_bwd_fused<8>(x, g, rstd, dy, residual, dx, dg, T, s);
    case 4096:
      if (norm_rows_off()) return launch_rmsnorm_bwd_fused<16>(x, g, rstd, dy, residual, dx, dg, T, s);
      if (!norm_batch_wait()) {
        launch_k(rmsnorm_bwd_pipe_kernel<16, 2>, dim3(std::max(1, std::min(num_sms(), (T + 1) / 2))), dim3(512), 0, s,
                 x, g, rstd, dy, residual, dx, dg, T);
        return status();
      }
      launch_k(rmsnorm_bwd_rows_kernel<16, 4>, dim3(std::max(1, std::min(num_sms(), (T + 3) / 4))), dim3(512), 0, s,
               x, g, rstd, dy, residual, dx, dg, T);
      return status();
    case 5120:
      if (!norm_batch_wait()) {
        launch_k(rmsnorm_bwd_pipe_kernel<20, 2>, dim3(std::max(1, std::min(num_sms(), (T + 1) / 2))), dim3(640), 0, s,
                 x, g, rstd, dy, residual, dx, dg, T);
        return status();
      }
      launch_k(rmsnorm_bwd_rows_kernel<20, 2>, dim3(std::max(1, std::min(2 * num_sms(), (T + 1) / 2))), dim3(640), 0, s,
               x, g, rstd, dy, residual, dx, dg, T);
      return status();
    default: break;
  }
  launch_k(rmsnorm_bwd_kernel, dim3(grid_for((T + 7) / 8)), dim3(kBlock), 0, s, x, g, rstd, dy, residual, dx, T, h);
  int rc = status();
  if (rc != PF_OK || dg == nullptr) return rc;
  // column blocks x row chunks so the grid covers ~2 waves
  const int col_blocks = (h + 255) / 256;
  int row_chunks = std::max(1, (2 * num_sms()) / col_blocks);
  const int rows_per_block = std::max(8, (T + row_chunks - 1) / row_chunks);
  row_chunks = (T + rows_per_block - 1) / rows_per_block;
  launch_k(rmsnorm_dg_kernel, dim3(dim3(col_blocks, row_chunks)), dim3(kBlock), 0, s, x, rstd, dy, dg, T, h, rows_per_block);
  return status();
}

int launch_rope_fwd(__nv_bfloat16* qkv, const float2* cs, int T, int seq, int nh, int nkv, int hd, cudaStream_t s) {
  if (hd % 16) return PF_ERR_INVALID;
  const int work = (nh + nkv) * (hd / 16);
  const int threads = std::min(kBlock, (work + 31) / 32 * 32);
  launch_k(rope_fwd_kernel, dim3(dim3((work + threads - 1) / threads, T)), dim3(threads), 0, s, qkv, cs, seq, nh, nkv, hd);
  return status();
}


int launch_swiglu_fwd(const __nv_bfloat16* gu, __nv_bfloat16* a, int T, int ffn, cudaStream_t s) {
  if (ffn % 128) return PF_ERR_INVALID;
  launch_k(swiglu_fwd_kernel, dim3(dim3((ffn / 8 + kBlock - 1) / kBlock, T)), dim3(kBlock), 0, s, gu, a, T, ffn);
  return status();
}

int launch_swiglu_bwd(const __nv_bfloat16* gu, const __nv_bfloat16* da, __nv_bfloat16* dgu, int T, int ffn,
                      cudaStream_t s) {
  if (ffn % 128) return PF_ERR_INVALID;
  launch_k(swiglu_bwd_kernel, dim3(dim3((ffn / 8 + kBlock - 1) / kBlock, T)), dim3(kBlock), 0, s, gu, da, dgu, T, ffn);
  return status();
}

int launch_cross_entropy(__nv_bfloat16* logits, const int* targets, float* loss_sum, int T, int V, float grad_scale,
                         float loss_scale, cudaStream_t s) {
  if (V % 8 || T <= 0) return PF_ERR_INVALID;
  if (V >= 16384)
    launch_k(cross_entropy_kernel<512>, dim3(T), dim3(512), 0, s, logits, targets, loss_sum, V, grad_scale,
             loss_scale);
  else
    launch_k(cross_entropy_kernel<kBlock>, dim3(T), dim3(kBlock), 0, s, logits, targets, loss_sum, V, grad_scale,
             loss_scale);
  return status();
}

int launch_init_normal(float* master, __nv_bfloat16* w, long long n, float stddev, uint64_t seed, cudaStream_t s) {
  if (n <= 0) return PF_OK;
  launch_k(init_normal_kernel, dim3(grid_for((n + kBlock - 1) / kBlock)), dim3(kBlock), 0, s, master, w, n, stddev, seed);
  return status();
}

int launch_fill(float* master, __nv_bfloat16* w, long long n, float v, cudaStream_t s) {
  if (n <= 0) return PF_OK;
  launch_k(fill_kernel, dim3(grid_for((n + kBlock - 1) / kBlock)), dim3(kBlock), 0, s, master, w, n, v);
  return status();
}

int launch_rope_table(float2* cs, int seq, int hd, float theta, cudaStream_t s) {
  launch_k(rope_table_kernel, dim3(grid_for((static_cast<long long>(seq) * hd / 2 + kBlock - 1) / kBlock)), dim3(kBlock), 0, s, 
      cs, seq, hd, theta);
  return status();
}

int launch_random_tokens(int* tok, long long n, int vocab, uint64_t seed, cudaStream_t s) {
  launch_k(random_tokens_kernel, dim3(grid_for((n + kBlock - 1) / kBlock)), dim3(kBlock), 0, s, tok, n, vocab, seed);
  return status();
}

}  // namespace pf
