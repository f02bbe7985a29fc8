// K3 on a CTA pair: the masked weight gradient over PAIRS of unfrozen 128x128 units.
//
//   G[u] (+)= dY[:, rows(u)]^T . X[:, cols(u)]      for every unfrozen unit u
//
// The pair MMA (tcgen05.mma.cta_group::2, M = 256, N = 128) multiplies a 256-row A
// held half in each CTA with ONE 128-column B split across the two CTAs, and
// leaves rows [128 r, 128 r + 128) in CTA r's TMEM. Two units that share their
// column block nb (the same X slice) but sit in any two row blocks therefore form
// one pair tile: CTA r stages its own unit's 128 dY columns and half of the shared
// X slice. Per SM and k-block that is 16 KB (A) + 8 KB (B) instead of the 1-CTA
// kernel's 16 + 16 KB for the same 128 x 128 x 64 of MMA work, which was the
// limiter of the 1-CTA dW (L2 -> SM operand traffic).
//
// Work lists come from K5p (mask_to_pairs_kernel): per matrix, groups of (band of
// 32 unit rows, column), each group's unfrozen units padded to an even count with
// -1. Entries (2i, 2i+1) are pair i. A -1 partner stages the leader's unit again
// (L2 hit) and skips its epilogue. Sweeping a band's columns in order keeps the
// band's dY columns in L2 while every X column block is read once per band. One
// launch covers up to kMaxDwProblems matrices (all of a stage's layers at once),
// so the launch's tail wave is a small fraction of it.
//
// The epilogue keeps K3's unit-stamp contract (gemm.cu): the first dW write of a
// unit in a step stores, later microbatches accumulate, and the stamp tells K6
// which units were touched (reference masked accumulation sum_m U_m . g_m,
// proj/src/sandbox.cpp:232-249; frozen units skipped, :250).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>

#include "kernels.cuh"
#include "pf_device_internal.hpp"
#include "kernel_util.cuh"
#include "ptx.cuh"

namespace pf {

int tma_desc_bf16_2d(CUtensorMap* map, const void* ptr, long long rows, long long cols, long long ld, int box_cols,
                     int box_rows);

namespace {

constexpr int BK = 64;
constexpr int STAGES = 8;
constexpr int A_BYTES = 128 * BK * 2;  // this CTA's unit: 128 dY columns x 64 tokens
constexpr int B_BYTES = 64 * BK * 2;   // this CTA's half of the shared X column block
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int TMEM_COLS = 256;  // two 128-column fp32 accumulators
constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + 1024;
constexpr int kEpiWarps = 4;
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr uint32_t IDESC = idesc_bf16_f32(256, 128, true, true);

struct alignas(64) DwProblem {
  CUtensorMap ta;  // dY stored [K][M] (MN-major A), box 64 x 64
  CUtensorMap tb;  // X  stored [K][N] (MN-major B), box 64 x 64
  float* C;
  long long ldc;
  const int* pairs;  // padded (band, column) unit list
  const int* count;  // device: padded entry count (even)
  int M, N, K;
  int tiles_n;
  int stamp_offset;
};

struct DwParams {
  DwProblem prob[kMaxDwProblems];
  int nprob;
  int* unit_stamp;
  int stamp;
};

// Smem table: prefix[i] = first pair index of problem i.
struct DwShared {
  int prefix[kMaxDwProblems + 1];
};

__device__ __forceinline__ int find_problem(const int* prefix, int nprob, int t) {
  int lo = 0, hi = nprob - 1;
  while (lo < hi) {  // last problem with prefix <= t
    const int mid = (lo + hi + 1) >> 1;
    if (prefix[mid] <= t) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm_dw_pair_kernel(const __grid_constant__ DwParams p) {
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
  __shared__ DwShared tab;

  const int warp = static_cast<int>(warp_uniform(threadIdx.x >> 5));  // uniform: MMA issue stays on the uniform datapath
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1;
  const int nclusters = gridDim.x >> 1;

  pdl_wait();  // the pair counts and operands come from the preceding kernels
  // pair counts of every problem -> prefix table (identical in both CTAs)
  if (threadIdx.x < p.nprob) tab.prefix[threadIdx.x + 1] = __ldcg(p.prob[threadIdx.x].count) >> 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 2 * 32 * kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc_pair(tmem_slot, TMEM_COLS);
    tmem_relinquish_pair();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    tab.prefix[0] = 0;
    for (int i = 0; i < p.nprob; ++i) tab.prefix[i + 1] += tab.prefix[i];
  }
  tc_fence_before();
  cluster_sync_all();  // barrier inits, TMEM allocation and the table visible
  tc_fence_after();
  const uint32_t tmem_base = warp_uniform(*tmem_slot);
  const int total = tab.prefix[p.nprob];

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------- producer (both CTAs)
      int stage = 0;
      uint32_t phase = 0;
      // the next item's pair entries are loaded one item ahead, off the TMA issue path
      auto load_pair = [&](int t) -> int2 {
        if (t >= total) return make_int2(0, 0);
        const int pi = find_problem(tab.prefix, p.nprob, t);
        const int li = t - tab.prefix[pi];
        return __ldg(reinterpret_cast<const int2*>(p.prob[pi].pairs) + li);
      };
      int2 nxt = load_pair(cluster);
      for (int t = cluster; t < total; t += nclusters) {
        const int pi = find_problem(tab.prefix, p.nprob, t);
        const DwProblem& pr = p.prob[pi];
        const int u0 = nxt.x, u1 = nxt.y;
        nxt = load_pair(t + nclusters);
        const int mine = (rank == 0 || u1 < 0) ? u0 : u1;
        const int mb = mine / pr.tiles_n;
        const int nb = u0 - (u0 / pr.tiles_n) * pr.tiles_n;
        const int num_kb = (pr.K + BK - 1) / BK;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * STAGE_BYTES);
          uint8_t* a_dst = sA + stage * A_BYTES;
          uint8_t* b_dst = sB + stage * B_BYTES;
          tma_load_2d_pair(a_dst, &pr.ta, &full_bar[stage], mb * 128, kb * BK);
          tma_load_2d_pair(a_dst + 8192, &pr.ta, &full_bar[stage], mb * 128 + 64, kb * BK);
          tma_load_2d_pair(b_dst, &pr.tb, &full_bar[stage], nb * 128 + static_cast<int>(rank) * 64, kb * BK);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      pdl_trigger();  // every load issued: the next kernel may launch (it waits for our completion)
    }
  } else if (warp == 1) {
    if (leader) {
      // ---------------------------------------------------------- MMA issuer (leader CTA; whole warp, one elected lane issues)
      int stage = 0;
      uint32_t phase = 0;
      int abuf = 0;
      uint32_t aphase = 0;
      for (int t = cluster; t < total; t += nclusters) {
        const int pi = find_problem(tab.prefix, p.nprob, t);
        const int num_kb = static_cast<int>(warp_uniform((p.prob[pi].K + BK - 1) / BK));
        mbar_wait(&tempty_bar[abuf], aphase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(abuf * 128);
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + stage * A_BYTES);
          const uint32_t b_base = smem_u32(sB + stage * B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // MN-major: advance 16 token rows = 2 swizzle atoms of 8 rows x 128 B
            const uint64_t adesc = sdesc_sw128(a_base + k * 2048, 8192, 1024);
            const uint64_t bdesc = sdesc_sw128(b_base + k * 2048, 8192, 1024);
            umma_bf16_pair_w(d_tmem, adesc, bdesc, IDESC, (kb | k) != 0 ? 1u : 0u);
          }
          umma_commit_pair_multicast_w(&empty_bar[stage], 0x3);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_pair_multicast_w(&tfull_bar[abuf], 0x3);
        abuf ^= 1;
        if (abuf == 0) aphase ^= 1;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row = q * 32 + static_cast<int>(lane);
    const uint32_t leader_tempty0 = mapa_shared(smem_u32(&tempty_bar[0]), 0);
    const uint32_t leader_tempty1 = mapa_shared(smem_u32(&tempty_bar[1]), 0);
    int abuf = 0;
    uint32_t aphase = 0;
    for (int t = cluster; t < total; t += nclusters) {
      const int pi = find_problem(tab.prefix, p.nprob, t);
      const DwProblem& pr = p.prob[pi];
      const int li = t - tab.prefix[pi];
      const int mine = __ldg(pr.pairs + 2 * li + static_cast<int>(rank));
      int unit = 0;
      bool first_touch = false;
      if (mine >= 0) {
        unit = pr.stamp_offset + mine;
        first_touch = __ldcg(p.unit_stamp + unit) != p.stamp;
      }
      mbar_wait(&tfull_bar[abuf], aphase);
      tc_fence_after();
      if (mine >= 0) {
        const int mb = mine / pr.tiles_n;
        const int nb = mine - mb * pr.tiles_n;
        const long long grow = static_cast<long long>(mb) * 128 + row;
        const bool row_ok = grow < pr.M;
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) +
                                 static_cast<uint32_t>(abuf * 128 + c * 32),
                             r);
          tmem_ld_wait();
          const int gcol = nb * 128 + c * 32;
          if (!row_ok || gcol >= pr.N) continue;
          float* cp = pr.C + grow * pr.ldc + gcol;
          if (gcol + 32 <= pr.N) {
            float4* c4 = reinterpret_cast<float4*>(cp);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              float4 w = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                     __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
              if (!first_touch) {
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
              if (gcol + i < pr.N) cp[i] = first_touch ? __uint_as_float(r[i]) : cp[i] + __uint_as_float(r[i]);
          }
        }
      }
      tc_fence_before();
      mbar_arrive_cluster(abuf ? leader_tempty1 : leader_tempty0);
      if (mine >= 0) {
        named_bar_sync(1, 32 * kEpiWarps);
        if (threadIdx.x == 64) p.unit_stamp[unit] = p.stamp;
      }
      abuf ^= 1;
      if (abuf == 0) aphase ^= 1;
    }
  }

  tc_fence_before();
  cluster_sync_all();  // both CTAs done with TMEM and with each other's barriers
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, TMEM_COLS);
  }
}

int max_dw_clusters() {
  static int n = -1;
  if (n < 0) {
    cudaFuncSetAttribute(gemm_dw_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * (num_sms() / 2));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = SMEM_BYTES;
    cudaLaunchAttribute attr{};
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = 2;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int c = 0;
    if (cudaOccupancyMaxActiveClusters(&c, gemm_dw_pair_kernel, &cfg) != cudaSuccess || c <= 0) {
      cudaGetLastError();
      c = num_sms() / 2;
    }
    n = std::min(c, num_sms() / 2);
  }
  return n;
}

// ---------------------------------------------------------------------------------------------
// Dense cells (gemm_dw_dense): a microbatch cell with no frozen unit -- the LP's plans are mostly
// 0 / 1 per cell -- needs every unit of every matrix, so its dW runs as whole 256 x 256 CTA-pair
// tiles (tcgen05.mma.cta_group::2, M = 256 = unit rows 2i, 2i + 1, one per CTA; N = 256 = unit
// columns 2j, 2j + 1, split across the pair's shared memory). Per SM and 16-token k-step the MMA
// reads 4 KB of A and 4 KB of its B half for 128 x 256 x 16 of work: the operand reuse of the
// forward / dX GEMMs, against 4 + 8 KB for the 1-CTA row-pair tile (shared-memory bound at ~0.67
// of the tensor pipe in the dense 8B launches, profiles/r2_bench_launches_fullstep.md). Edge
// units past M / N read TMA zero fill and are skipped by the epilogue. Same unit-stamp contract.
constexpr int Q_STAGES = 6;
constexpr int QB_BYTES = 128 * BK * 2;  // this CTA's 128 of the tile's 256 X columns
constexpr int Q_STAGE_BYTES = A_BYTES + QB_BYTES;
constexpr int Q_SMEM_BYTES = 1024 + Q_STAGES * Q_STAGE_BYTES + 1024;
constexpr uint32_t IDESC_Q = idesc_bf16_f32(256, 256, true, true);

struct DenseParams {
  DwProblem prob[kMaxDwProblems];
  int prefix[kMaxDwProblems + 1];  // first quad of problem i (host-computed)
  unsigned char rows_fast[kMaxDwProblems];
  int nprob;
  int* unit_stamp;
  int stamp;
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm_dw_quad_kernel(const __grid_constant__ DenseParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + Q_STAGES * A_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + Q_STAGES * Q_STAGE_BYTES);
  uint64_t* empty_bar = full_bar + Q_STAGES;
  uint64_t* tfull_bar = empty_bar + Q_STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = static_cast<int>(warp_uniform(threadIdx.x >> 5));
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1;
  const int nclusters = gridDim.x >> 1;
  const int total = p.prefix[p.nprob];

  pdl_wait();
  if (threadIdx.x == 0) {
    for (int s = 0; s < Q_STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 2 * 32 * kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc_pair(tmem_slot, 512);
    tmem_relinquish_pair();
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = warp_uniform(*tmem_slot);

  // quad t -> (problem, unit row pair, unit column pair)
  auto quad = [&](int t, int& pi, int& mrow, int& mcol) {
    int lo = 0, hi = p.nprob - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (p.prefix[mid] <= t) lo = mid;
      else hi = mid - 1;
    }
    pi = lo;
    const int q = t - p.prefix[pi];
    if (p.rows_fast[pi]) {  // dY (T x M) is the smaller operand: sweep the unit-row pairs of a column
      const int qm = (((p.prob[pi].M + 127) >> 7) + 1) >> 1;  // pair first, so X streams from DRAM once
      mcol = q / qm;
      mrow = q - mcol * qm;
    } else {
      const int qn = (p.prob[pi].tiles_n + 1) >> 1;
      mrow = q / qn;
      mcol = q - mrow * qn;
    }
  };

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------- producer (both CTAs)
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cluster; t < total; t += nclusters) {
        int pi, mrow, mcol;
        quad(t, pi, mrow, mcol);
        const DwProblem& pr = p.prob[pi];
        const int mb = 2 * mrow + static_cast<int>(rank);
        const int nb = 2 * mcol + static_cast<int>(rank);
        const int num_kb = (pr.K + BK - 1) / BK;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * Q_STAGE_BYTES);
          uint8_t* a_dst = sA + stage * A_BYTES;
          uint8_t* b_dst = sB + stage * QB_BYTES;
          tma_load_2d_pair(a_dst, &pr.ta, &full_bar[stage], mb * 128, kb * BK);
          tma_load_2d_pair(a_dst + 8192, &pr.ta, &full_bar[stage], mb * 128 + 64, kb * BK);
          tma_load_2d_pair(b_dst, &pr.tb, &full_bar[stage], nb * 128, kb * BK);
          tma_load_2d_pair(b_dst + 8192, &pr.tb, &full_bar[stage], nb * 128 + 64, kb * BK);
          if (++stage == Q_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      pdl_trigger();
    }
  } else if (warp == 1) {
    if (leader) {
      // ---------------------------------------------------------- MMA issuer (leader CTA)
      int stage = 0;
      uint32_t phase = 0;
      int abuf = 0;
      uint32_t aphase = 0;
      for (int t = cluster; t < total; t += nclusters) {
        int pi, mrow, mcol;
        quad(t, pi, mrow, mcol);
        const int num_kb = static_cast<int>(warp_uniform((p.prob[pi].K + BK - 1) / BK));
        mbar_wait(&tempty_bar[abuf], aphase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(abuf * 256);
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + stage * A_BYTES);
          const uint32_t b_base = smem_u32(sB + stage * QB_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t adesc = sdesc_sw128(a_base + k * 2048, 8192, 1024);
            const uint64_t bdesc = sdesc_sw128(b_base + k * 2048, 8192, 1024);
            umma_bf16_pair_w(d_tmem, adesc, bdesc, IDESC_Q, (kb | k) != 0 ? 1u : 0u);
          }
          umma_commit_pair_multicast_w(&empty_bar[stage], 0x3);
          if (++stage == Q_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_pair_multicast_w(&tfull_bar[abuf], 0x3);
        abuf ^= 1;
        if (abuf == 0) aphase ^= 1;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (both CTAs): this CTA's
    // unit row, units (mb, 2 mcol) and (mb, 2 mcol + 1)
    const int q = warp & 3;
    const int row = q * 32 + static_cast<int>(lane);
    const uint32_t leader_tempty0 = mapa_shared(smem_u32(&tempty_bar[0]), 0);
    const uint32_t leader_tempty1 = mapa_shared(smem_u32(&tempty_bar[1]), 0);
    int abuf = 0;
    uint32_t aphase = 0;
    for (int t = cluster; t < total; t += nclusters) {
      int pi, mrow, mcol;
      quad(t, pi, mrow, mcol);
      const DwProblem& pr = p.prob[pi];
      const int mb = 2 * mrow + static_cast<int>(rank);
      const int tiles_m = (pr.M + 127) >> 7;
      const bool row_unit = mb < tiles_m;
      const int nb0 = 2 * mcol;
      const bool has1 = nb0 + 1 < pr.tiles_n;
      const int u0 = mb * pr.tiles_n + nb0;
      const bool first0 = row_unit && __ldcg(p.unit_stamp + pr.stamp_offset + u0) != p.stamp;
      const bool first1 = row_unit && has1 && __ldcg(p.unit_stamp + pr.stamp_offset + u0 + 1) != p.stamp;
      mbar_wait(&tfull_bar[abuf], aphase);
      tc_fence_after();
      const long long grow = static_cast<long long>(mb) * 128 + row;
      const bool row_ok = row_unit && grow < pr.M;
#pragma unroll 1
      for (int c = 0; c < 8; ++c) {
        if (c >= 4 && !has1) break;
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(abuf * 256 + c * 32),
                           r);
        tmem_ld_wait();
        const int gcol = nb0 * 128 + c * 32;
        const bool first = c < 4 ? first0 : first1;
        if (!row_ok || gcol >= pr.N) continue;
        float* cp = pr.C + grow * pr.ldc + gcol;
        if (gcol + 32 <= pr.N) {
          float4* c4 = reinterpret_cast<float4*>(cp);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float4 w = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]), __uint_as_float(r[4 * j + 2]),
                                   __uint_as_float(r[4 * j + 3]));
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
      mbar_arrive_cluster(abuf ? leader_tempty1 : leader_tempty0);
      if (row_unit) {
        named_bar_sync(1, 32 * kEpiWarps);
        if (threadIdx.x == 64) {
          p.unit_stamp[pr.stamp_offset + u0] = p.stamp;
          if (has1) p.unit_stamp[pr.stamp_offset + u0 + 1] = p.stamp;
        }
      }
      abuf ^= 1;
      if (abuf == 0) aphase ^= 1;
    }
  }

  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, 512);
  }
}

}  // namespace

int gemm_dw_pairs(const DwGemm* items, int n, int* unit_stamp, int stamp, cudaStream_t stream) {
  if (n < 0 || unit_stamp == nullptr) return PF_ERR_INVALID;
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(gemm_dw_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES) !=
        cudaSuccess)
      return PF_ERR_CUDA;
    attr_set = true;
  }
  for (int base = 0; base < n; base += kMaxDwProblems) {
    const int cnt = std::min(kMaxDwProblems, n - base);
    DwParams p{};
    p.nprob = cnt;
    p.unit_stamp = unit_stamp;
    p.stamp = stamp;
    long long max_pairs = 0;
    for (int i = 0; i < cnt; ++i) {
      const DwGemm& it = items[base + i];
      if (it.M <= 0 || it.N <= 0 || it.K <= 0 || (it.K % 8) != 0 || !it.list || !it.count || !it.C)
        return PF_ERR_INVALID;
      DwProblem& pr = p.prob[i];
      if (int rc = tma_desc_bf16_2d(&pr.ta, it.dy, it.K, it.M, it.ldy, 64, 64)) return rc;
      if (int rc = tma_desc_bf16_2d(&pr.tb, it.x, it.K, it.N, it.ldx, 64, 64)) return rc;
      pr.C = it.C;
      pr.ldc = it.ldc;
      pr.pairs = it.list;
      pr.count = it.count;
      pr.M = it.M;
      pr.N = it.N;
      pr.K = it.K;
      pr.tiles_n = (it.N + 127) / 128;
      pr.stamp_offset = it.stamp_offset;
      const int tiles_m = (it.M + 127) / 128;
      max_pairs += (static_cast<long long>(tiles_m) * pr.tiles_n + pair_groups(tiles_m, pr.tiles_n)) / 2;
    }
    const int clusters = static_cast<int>(std::min<long long>(max_pairs, max_dw_clusters()));
    if (clusters <= 0) continue;
    launch_k(gemm_dw_pair_kernel, dim3(2 * clusters), dim3(kThreads), SMEM_BYTES, stream, p);
    count_launch();
    if (cudaPeekAtLastError() != cudaSuccess) return PF_ERR_CUDA;
  }
  return PF_OK;
}

int gemm_dw_dense(const DwGemm* items, int n, int* unit_stamp, int stamp, cudaStream_t stream) {
  if (n < 0 || unit_stamp == nullptr) return PF_ERR_INVALID;
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(gemm_dw_quad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, Q_SMEM_BYTES) !=
        cudaSuccess)
      return PF_ERR_CUDA;
    attr_set = true;
  }
  for (int base = 0; base < n; base += kMaxDwProblems) {
    const int cnt = std::min(kMaxDwProblems, n - base);
    DenseParams p{};
    p.nprob = cnt;
    p.unit_stamp = unit_stamp;
    p.stamp = stamp;
    p.prefix[0] = 0;
    for (int i = 0; i < cnt; ++i) {
      const DwGemm& it = items[base + i];
      if (it.M <= 0 || it.N <= 0 || it.K <= 0 || (it.K % 8) != 0 || !it.C) return PF_ERR_INVALID;
      DwProblem& pr = p.prob[i];
      if (int rc = tma_desc_bf16_2d(&pr.ta, it.dy, it.K, it.M, it.ldy, 64, 64)) return rc;
      if (int rc = tma_desc_bf16_2d(&pr.tb, it.x, it.K, it.N, it.ldx, 64, 64)) return rc;
      pr.C = it.C;
      pr.ldc = it.ldc;
      pr.M = it.M;
      pr.N = it.N;
      pr.K = it.K;
      pr.tiles_n = (it.N + 127) / 128;
      pr.stamp_offset = it.stamp_offset;
      const int tiles_m = (it.M + 127) / 128;
      p.prefix[i + 1] = p.prefix[i] + ((tiles_m + 1) / 2) * ((pr.tiles_n + 1) / 2);
      p.rows_fast[i] = it.M <= it.N ? 1 : 0;
    }
    const int clusters = std::min(p.prefix[cnt], num_sms() / 2);
    if (clusters <= 0) continue;
    launch_k(gemm_dw_quad_kernel, dim3(2 * clusters), dim3(kThreads), Q_SMEM_BYTES, stream, p);
    count_launch();
    if (cudaPeekAtLastError() != cudaSuccess) return PF_ERR_CUDA;
  }
  return PF_OK;
}

}  // namespace pf
