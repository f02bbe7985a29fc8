// K3 over ROW PAIRS of unfrozen 128x128 units: one CTA computes two units of the same
// weight row block, G[mb][nb0] and G[mb][nb1], with one 128 x 256 x 16 MMA per K step:
//
//   D[128, 256] = dY[:, rows mb]^T . [X[:, cols nb0] | X[:, cols nb1]]
//
// The shared operand (the unit row's dY block) is read from shared memory once per 256
// output columns instead of once per 128: per 128-column unit and K step the MMA reads
// 4 + 8 KB for two units instead of 2 x (4 + 4) KB, and TMA writes 3/4 of the bytes (the
// 1-CTA 128 x 128 unit tile is bound by shared-memory bandwidth at ~50% of the tensor pipe,
// profiles/r1_dw_bench.txt). A row with an odd unfrozen count ends with a single unit
// (N = 128 MMA) -- no padding work. Work lists come from K5r (mask_to_rowpairs_kernel).
//
// The epilogue keeps K3's unit-stamp contract (gemm.cu): the first dW write of a unit in
// a step stores, later microbatches accumulate, the stamp tells K6 which units were touched
// (reference masked accumulation sum_m U_m . g_m, proj/src/sandbox.cpp:232-249).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>

#include "kernel_util.cuh"
#include "kernels.cuh"
#include "pf_device_internal.hpp"
#include "ptx.cuh"

namespace pf {

int tma_desc_bf16_2d(CUtensorMap* map, const void* ptr, long long rows, long long cols, long long ld, int box_cols,
                     int box_rows);

namespace {

constexpr int BK = 64;
constexpr int STAGES = 4;
constexpr int A_BYTES = 128 * BK * 2;  // the unit row's dY block: 128 columns x 64 tokens
constexpr int B_BYTES = 256 * BK * 2;  // X blocks of the two units: 2 x 128 columns x 64 tokens
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int TMEM_COLS = 512;  // two 256-column fp32 accumulators
constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + 256;
constexpr int kThreads = 192;
constexpr uint32_t IDESC_PAIR = idesc_bf16_f32(128, 256, true, true);
constexpr uint32_t IDESC_ONE = idesc_bf16_f32(128, 128, true, true);

struct alignas(64) RowProblem {
  CUtensorMap ta;  // dY stored [K][M] (MN-major A), box 64 x 64
  CUtensorMap tb;  // X  stored [K][N] (MN-major B), box 64 x 64
  float* C;
  long long ldc;
  const int2* list;  // K5r entries {u0, u1 or -1}, same row block
  const int* count;  // device: entry count
  int M, N, K;
  int tiles_n;
  int stamp_offset;
};

struct RowParams {
  RowProblem prob[kMaxDwProblems];
  int nprob;
  int* unit_stamp;
  int stamp;
};

__device__ __forceinline__ int find_problem(const int* prefix, int nprob, int t) {
  int lo = 0, hi = nprob - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (prefix[mid] <= t) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(kThreads, 1) gemm_dw_rowpair_kernel(const __grid_constant__ RowParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  __shared__ int prefix[kMaxDwProblems + 1];

  const int warp = static_cast<int>(warp_uniform(threadIdx.x >> 5));  // uniform: MMA issue stays on the uniform datapath
  const uint32_t lane = threadIdx.x & 31;

  pdl_wait();  // entry counts and operands come from the preceding kernels
  if (threadIdx.x < p.nprob) prefix[threadIdx.x + 1] = __ldcg(p.prob[threadIdx.x].count);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 128);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane < static_cast<uint32_t>(p.nprob)) {
    tma_prefetch(&p.prob[lane].ta);
    tma_prefetch(&p.prob[lane].tb);
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, TMEM_COLS);
    tmem_relinquish();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    prefix[0] = 0;
    for (int i = 0; i < p.nprob; ++i) prefix[i + 1] += prefix[i];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = warp_uniform(*tmem_slot);
  const int total = prefix[p.nprob];

  auto entry = [&](int t, int& pi) -> int2 {
    pi = find_problem(prefix, p.nprob, t);
    return __ldg(p.prob[pi].list + (t - prefix[pi]));
  };

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ producer
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        int pi;
        const int2 e = entry(t, pi);
        const RowProblem& pr = p.prob[pi];
        const int mb = e.x / pr.tiles_n;
        const int nb0 = e.x - mb * pr.tiles_n;
        const int nb1 = e.y >= 0 ? e.y - mb * pr.tiles_n : -1;
        const uint32_t bytes = A_BYTES + (nb1 >= 0 ? B_BYTES : B_BYTES / 2);
        const int num_kb = (pr.K + BK - 1) / BK;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full_bar[stage], bytes);
          uint8_t* a_dst = sA + stage * A_BYTES;
          uint8_t* b_dst = sB + stage * B_BYTES;
          tma_load_2d(a_dst, &pr.ta, &full_bar[stage], mb * 128, kb * BK);
          tma_load_2d(a_dst + 8192, &pr.ta, &full_bar[stage], mb * 128 + 64, kb * BK);
          tma_load_2d(b_dst, &pr.tb, &full_bar[stage], nb0 * 128, kb * BK);
          tma_load_2d(b_dst + 8192, &pr.tb, &full_bar[stage], nb0 * 128 + 64, kb * BK);
          if (nb1 >= 0) {
            tma_load_2d(b_dst + 16384, &pr.tb, &full_bar[stage], nb1 * 128, kb * BK);
            tma_load_2d(b_dst + 24576, &pr.tb, &full_bar[stage], nb1 * 128 + 64, kb * BK);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      pdl_trigger();
    }
  } else if (warp == 1) {
    {
      // ------------------------------------------------------------ MMA issuer (whole warp, one elected lane issues)
      int stage = 0;
      uint32_t phase = 0;
      int abuf = 0;
      uint32_t aphase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        int pi;
        const int2 e = entry(t, pi);
        const uint32_t idesc = warp_uniform(e.y >= 0 ? IDESC_PAIR : IDESC_ONE);
        const int num_kb = static_cast<int>(warp_uniform((p.prob[pi].K + BK - 1) / BK));
        mbar_wait(&tempty_bar[abuf], aphase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(abuf * 256);
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + stage * A_BYTES);
          const uint32_t b_base = smem_u32(sB + stage * B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // MN-major: 16 token rows = 2 swizzle atoms of 8 rows x 128 B; 64-column chunks 8 KB apart
            const uint64_t adesc = sdesc_sw128(a_base + k * 2048, 8192, 1024);
            const uint64_t bdesc = sdesc_sw128(b_base + k * 2048, 8192, 1024);
            umma_bf16_w(d_tmem, adesc, bdesc, idesc, (kb | k) != 0 ? 1u : 0u);
          }
          umma_commit_w(&empty_bar[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_w(&tfull_bar[abuf]);
        abuf ^= 1;
        if (abuf == 0) aphase ^= 1;
      }
    }
  } else {
    // -------------------------------------------------------------- epilogue
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row = q * 32 + static_cast<int>(lane);
    int abuf = 0;
    uint32_t aphase = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      int pi;
      const int2 e = entry(t, pi);
      const RowProblem& pr = p.prob[pi];
      const int mb = e.x / pr.tiles_n;
      const int units = e.y >= 0 ? 2 : 1;
      const bool first0 = __ldcg(p.unit_stamp + pr.stamp_offset + e.x) != p.stamp;
      const bool first1 = units == 2 && __ldcg(p.unit_stamp + pr.stamp_offset + e.y) != p.stamp;
      mbar_wait(&tfull_bar[abuf], aphase);
      tc_fence_after();
      const long long grow = static_cast<long long>(mb) * 128 + row;
      const bool row_ok = grow < pr.M;
#pragma unroll 1
      for (int c = 0; c < 4 * units; ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) +
                               static_cast<uint32_t>(abuf * 256 + c * 32),
                           r);
        tmem_ld_wait();
        const int u = c < 4 ? e.x : e.y;
        const bool first = c < 4 ? first0 : first1;
        const int gcol = (u - mb * pr.tiles_n) * 128 + (c & 3) * 32;
        if (!row_ok || gcol >= pr.N) continue;
        float* cp = pr.C + grow * pr.ldc + gcol;
        if (gcol + 32 <= pr.N) {
          float4* c4 = reinterpret_cast<float4*>(cp);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float4 w = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                   __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
            if (!first) {
              const float4 o = c4[j];
              w.x += o.x;
              w.y += o.y;
              w.z += o.z;
              w.w += o.w;
            }
            c4[j] = w;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (gcol + i < pr.N) cp[i] = first ? __uint_as_float(r[i]) : cp[i] + __uint_as_float(r[i]);
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty_bar[abuf]);
      named_bar_sync(1, 128);
      if (threadIdx.x == 64) {
        p.unit_stamp[pr.stamp_offset + e.x] = p.stamp;
        if (units == 2) p.unit_stamp[pr.stamp_offset + e.y] = p.stamp;
      }
      abuf ^= 1;
      if (abuf == 0) aphase ^= 1;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

}  // namespace

int gemm_dw_rowpairs(const DwGemm* items, int n, int* unit_stamp, int stamp, cudaStream_t stream) {
  if (n < 0 || unit_stamp == nullptr) return PF_ERR_INVALID;
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(gemm_dw_rowpair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES) !=
        cudaSuccess)
      return PF_ERR_CUDA;
    attr_set = true;
  }
  for (int base = 0; base < n; base += kMaxDwProblems) {
    const int cnt = std::min(kMaxDwProblems, n - base);
    RowParams p{};
    p.nprob = cnt;
    p.unit_stamp = unit_stamp;
    p.stamp = stamp;
    long long max_entries = 0;
    for (int i = 0; i < cnt; ++i) {
      const DwGemm& it = items[base + i];
      if (it.M <= 0 || it.N <= 0 || it.K <= 0 || (it.K % 8) != 0 || !it.list || !it.count || !it.C)
        return PF_ERR_INVALID;
      RowProblem& pr = p.prob[i];
      if (int rc = tma_desc_bf16_2d(&pr.ta, it.dy, it.K, it.M, it.ldy, 64, 64)) return rc;
      if (int rc = tma_desc_bf16_2d(&pr.tb, it.x, it.K, it.N, it.ldx, 64, 64)) return rc;
      pr.C = it.C;
      pr.ldc = it.ldc;
      pr.list = reinterpret_cast<const int2*>(it.list);
      pr.count = it.count;
      pr.M = it.M;
      pr.N = it.N;
      pr.K = it.K;
      pr.tiles_n = (it.N + 127) / 128;
      pr.stamp_offset = it.stamp_offset;
      const int tiles_m = (it.M + 127) / 128;
      max_entries += (static_cast<long long>(tiles_m) * pr.tiles_n + tiles_m) / 2;
    }
    const int grid = static_cast<int>(std::min<long long>(max_entries, num_sms()));
    if (grid <= 0) continue;
    launch_k(gemm_dw_rowpair_kernel, dim3(grid), dim3(kThreads), SMEM_BYTES, stream, p);
    count_launch();
    if (cudaPeekAtLastError() != cudaSuccess) return PF_ERR_CUDA;
  }
  return PF_OK;
}

}  // namespace pf
