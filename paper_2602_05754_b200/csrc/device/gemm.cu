// K1 / K2 / K3: persistent warp-specialized tcgen05 GEMM for sm_100a.
//
//   C[M,N] (op)= alpha * A[M,K] . B[N,K]^T      bf16 in, fp32 accumulate in TMEM
//
// A and B are each either K-major (row-major [rows][K]) or MN-major (row-major
// [K][rows]); the MMA consumes both straight from SWIZZLE_128B shared memory,
// so the three training GEMMs need no transposes:
//   forward  Y  = X  . W^T      A = X  (K-major)  B = W (K-major)
//   dX       dX = dY . W        A = dY (K-major)  B = W (MN-major)
//   dW       dW = dY^T . X      A = dY (MN-major) B = X (MN-major)
// The dW launch runs over device-resident work lists of unfrozen 128x128 units
// (K5 output) of up to kMaxProblems weight matrices at once (grouped, so a
// layer's four matrices fill the GPU together), so its time is linear in the
// unfrozen count: the device realisation of w = w_max - r (w_max - w_min)
// (reference proj/src/timing.cpp:53) and of the masked accumulation
// sum_m U_m . g_m (reference proj/src/sandbox.cpp:232-249).
//
// Roles (192 threads, 1 CTA per SM, persistent over tiles):
//   warp 0      TMA producer (one lane): smem ring of STAGES {A,B} k-blocks
//   warp 1      TMEM allocator + MMA issuer (one lane): tcgen05.mma into a
//               double-buffered TMEM accumulator (2 x BN fp32 columns)
//   warps 2..5  epilogue: tcgen05.ld -> registers -> global (bf16 / fp32)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <mutex>

#include "kernel_util.cuh"
#include "ptx.cuh"
#include "pf_device_internal.hpp"

namespace pf {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // one 128-byte swizzle span of bf16
constexpr int GROUP_M = 16;
constexpr int kThreads = 192;

template <int BN>
struct GemmCfg {
  static constexpr int STAGES = BN == 256 ? 4 : 6;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + 256;
};

struct alignas(64) Problem {
  CUtensorMap ta;  // A operand (TMA descriptor, lives in kernel-parameter space)
  CUtensorMap tb;  // B operand
  void* C;
  long long ldc;
  int M, N;
  int tiles_m, tiles_n;
  const int* list;   // list mode: local unit ids (mb * tiles_n + nb)
  const int* count;  // list mode: device-resident count
  int stamp_offset;  // first global unit id of this matrix (EPI_ACC_F32)
  int num_tiles;     // plain mode
  int num_kb;        // k-blocks of this problem (list mode: K differs per matrix)
};

// MAXP = 1 for one plain GEMM; kMaxDwProblems for the batched masked dW (list mode), whose
// parameter block holds every matrix of a microbatch (<= 32 KB of kernel parameters).
template <int MAXP>
struct GemmParams {
  Problem prob[MAXP];
  int nprob;
  float alpha;
  int list_mode;
  int* unit_stamp;  // EPI_ACC_F32 first-touch stamps
  int stamp;
};

// prefix[i] = first tile of problem i (shared memory, filled once per CTA)
template <int MAXP>
__device__ __forceinline__ int find_prob(const int* prefix, int nprob, int t) {
  if constexpr (MAXP == 1) {
    return 0;
  } else {
    int lo = 0, hi = nprob - 1;
    while (lo < hi) {  // last problem with prefix <= t
      const int mid = (lo + hi + 1) >> 1;
      if (prefix[mid] <= t) lo = mid;
      else hi = mid - 1;
    }
    return lo;
  }
}

// unit entry of tile t (list mode) or -1 (plain mode / past the end)
template <int MAXP>
__device__ __forceinline__ int tile_unit(const GemmParams<MAXP>& p, const int* prefix, int total, int t) {
  if (!p.list_mode || t >= total) return -1;
  const int pi = find_prob<MAXP>(prefix, p.nprob, t);
  return __ldg(p.prob[pi].list + (t - prefix[pi]));
}

template <int MAXP>
__device__ __forceinline__ void decode_tile(const GemmParams<MAXP>& p, const int* prefix, int t, int unit, int& pi,
                                            int& mb, int& nb) {
  pi = find_prob<MAXP>(prefix, p.nprob, t);
  const Problem& pr = p.prob[pi];
  const int lt = t - prefix[pi];
  if (p.list_mode) {
    mb = unit / pr.tiles_n;
    nb = unit - mb * pr.tiles_n;
    return;
  }
  const int group_size = GROUP_M * pr.tiles_n;
  const int g = lt / group_size;
  const int first_m = g * GROUP_M;
  const int gm = min(pr.tiles_m - first_m, GROUP_M);
  const int local = lt - g * group_size;
  mb = first_m + local % gm;
  nb = local / gm;
}

template <int BN, bool A_MN, bool B_MN, int EPI, int MAXP>
__global__ void __launch_bounds__(kThreads, 1) gemm_tcgen05_kernel(const __grid_constant__ GemmParams<MAXP> p) {
  using Cfg = GemmCfg<BN>;
  constexpr int STAGES = Cfg::STAGES;
  constexpr uint32_t IDESC = idesc_bf16_f32(BM, BN, A_MN, B_MN);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * Cfg::A_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = static_cast<int>(warp_uniform(threadIdx.x >> 5));  // uniform: MMA issue stays on the uniform datapath
  const uint32_t lane = threadIdx.x & 31;

  __shared__ int prefix[MAXP + 1];
  pdl_wait();  // the unit counts (and operands) come from the preceding kernels
  if (threadIdx.x < p.nprob)
    prefix[threadIdx.x + 1] = p.list_mode ? __ldcg(p.prob[threadIdx.x].count) : p.prob[threadIdx.x].num_tiles;

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
    tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
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
  const int ntiles = prefix[p.nprob];

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ producer
      int stage = 0;
      uint32_t phase = 0;
      // list mode: the next tile's unit id is loaded one tile ahead, off the TMA issue path
      int nxt = tile_unit(p, prefix, ntiles, blockIdx.x);
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int pi, mb, nb;
        decode_tile(p, prefix, t, nxt, pi, mb, nb);
        nxt = tile_unit(p, prefix, ntiles, t + gridDim.x);
        const CUtensorMap* ta = &p.prob[pi].ta;
        const CUtensorMap* tb = &p.prob[pi].tb;
        const int num_kb = p.prob[pi].num_kb;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full_bar[stage], Cfg::STAGE_BYTES);
          uint8_t* a_dst = sA + stage * Cfg::A_BYTES;
          uint8_t* b_dst = sB + stage * Cfg::B_BYTES;
          if constexpr (!A_MN) {
            tma_load_2d(a_dst, ta, &full_bar[stage], kb * BK, mb * BM);
          } else {
#pragma unroll
            for (int c = 0; c < BM / 64; ++c)
              tma_load_2d(a_dst + c * 8192, ta, &full_bar[stage], mb * BM + c * 64, kb * BK);
          }
          if constexpr (!B_MN) {
            tma_load_2d(b_dst, tb, &full_bar[stage], kb * BK, nb * BN);
          } else {
#pragma unroll
            for (int c = 0; c < BN / 64; ++c)
              tma_load_2d(b_dst + c * 8192, tb, &full_bar[stage], nb * BN + c * 64, kb * BK);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      pdl_trigger();  // every load issued: the next kernel may launch (it waits for our completion)
    }
  } else if (warp == 1) {
    {
      // ------------------------------------------------------------ MMA issuer (whole warp, one elected lane issues)
      int stage = 0;
      uint32_t phase = 0;
      int abuf = 0;
      uint32_t aphase = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int num_kb = static_cast<int>(warp_uniform(p.prob[find_prob<MAXP>(prefix, p.nprob, t)].num_kb));
        mbar_wait(&tempty_bar[abuf], aphase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(abuf * BN);
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + stage * Cfg::A_BYTES);
          const uint32_t b_base = smem_u32(sB + stage * Cfg::B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // K-major: advance 16 elements = 32 B inside the swizzle atom.
            // MN-major: advance 16 K-rows = 2 atoms of 8 rows x 128 B.
            const uint64_t adesc = A_MN ? sdesc_sw128(a_base + k * 2048, 8192, 1024)
                                        : sdesc_sw128(a_base + k * 32, 16, 1024);
            const uint64_t bdesc = B_MN ? sdesc_sw128(b_base + k * 2048, 8192, 1024)
                                        : sdesc_sw128(b_base + k * 32, 16, 1024);
            umma_bf16_w(d_tmem, adesc, bdesc, IDESC, (kb | k) != 0 ? 1u : 0u);
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
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      int pi, mb, nb;
      decode_tile(p, prefix, t, tile_unit(p, prefix, ntiles, t), pi, mb, nb);
      const Problem& pr = p.prob[pi];
      bool first_touch = false;
      int unit = 0;
      if constexpr (EPI == EPI_ACC_F32) {
        unit = pr.stamp_offset + mb * pr.tiles_n + nb;
        first_touch = p.unit_stamp[unit] != p.stamp;
      }
      mbar_wait(&tfull_bar[abuf], aphase);
      tc_fence_after();
      const long long grow = static_cast<long long>(mb) * BM + row;
      const bool row_ok = grow < pr.M;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) +
                               static_cast<uint32_t>(abuf * BN + c * 32),
                           r);
        tmem_ld_wait();
        const int gcol = nb * BN + c * 32;
        if (!row_ok || gcol >= pr.N) continue;
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]) * p.alpha;
        const bool full = gcol + 32 <= pr.N;
        if constexpr (EPI == EPI_STORE_BF16 || EPI == EPI_ADD_BF16) {
          __nv_bfloat16* cp = reinterpret_cast<__nv_bfloat16*>(pr.C) + grow * pr.ldc + gcol;
          if (full) {
            uint4* c4 = reinterpret_cast<uint4*>(cp);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              float w[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) w[i] = v[j * 8 + i];
              if constexpr (EPI == EPI_ADD_BF16) {
                const uint4 old = c4[j];
                const __nv_bfloat162* o = reinterpret_cast<const __nv_bfloat162*>(&old);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  const float2 f = __bfloat1622float2(o[i]);
                  w[2 * i] += f.x;
                  w[2 * i + 1] += f.y;
                }
              }
              uint4 out;
              out.x = pack_bf16x2(w[0], w[1]);
              out.y = pack_bf16x2(w[2], w[3]);
              out.z = pack_bf16x2(w[4], w[5]);
              out.w = pack_bf16x2(w[6], w[7]);
              c4[j] = out;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              if (gcol + i < pr.N) {
                float w = v[i];
                if constexpr (EPI == EPI_ADD_BF16) w += __bfloat162float(cp[i]);
                cp[i] = __float2bfloat16_rn(w);
              }
            }
          }
        } else {
          float* cp = reinterpret_cast<float*>(pr.C) + grow * pr.ldc + gcol;
          if (full) {
            float4* c4 = reinterpret_cast<float4*>(cp);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              float4 w = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
              if (EPI == EPI_ACC_F32 && !first_touch) {
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
            for (int i = 0; i < 32; ++i) {
              if (gcol + i < pr.N) {
                float w = v[i];
                if (EPI == EPI_ACC_F32 && !first_touch) w += cp[i];
                cp[i] = w;
              }
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty_bar[abuf]);
      if constexpr (EPI == EPI_ACC_F32) {
        named_bar_sync(1, 128);
        if (threadIdx.x == 64) p.unit_stamp[unit] = p.stamp;
      }
      abuf ^= 1;
      if (abuf == 0) aphase ^= 1;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

// Row-major bf16 matrix [rows][cols] with row stride ld (elements); box
// {box_cols (inner), box_rows}.
int make_tmap(CUtensorMap* map, const void* ptr, long long rows, long long cols, long long ld, int box_cols,
              int box_rows, CUtensorMapSwizzle swizzle = CU_TENSOR_MAP_SWIZZLE_128B) {
  auto encode = get_encode();
  if (!encode) return PF_ERR_CUDA;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 2)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  // invalid geometry (row stride not a multiple of 16 B, misaligned base, ...)
  return r == CUDA_SUCCESS ? PF_OK : PF_ERR_INVALID;
}

template <int BN, bool A_MN, bool B_MN, int EPI, int MAXP = 1>
int launch(const GemmParams<MAXP>& p, int grid_limit, cudaStream_t stream) {
  using Cfg = GemmCfg<BN>;
  auto kern = gemm_tcgen05_kernel<BN, A_MN, B_MN, EPI, MAXP>;
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES) != cudaSuccess)
      return PF_ERR_CUDA;
    attr_set = true;
  }
  const int grid = std::min(grid_limit, num_sms());
  if (grid <= 0) return PF_OK;
  launch_k(kern, dim3(grid), dim3(kThreads), Cfg::SMEM_BYTES, stream, p);
  count_launch();
  return cudaPeekAtLastError() == cudaSuccess ? PF_OK : PF_ERR_CUDA;
}

template <int BN>
int dispatch(bool a_mn, bool b_mn, const GemmParams<1>& p, int epi, int grid_limit, cudaStream_t s) {
  const int key = (a_mn ? 1 : 0) | (b_mn ? 2 : 0);
#define PF_GEMM_CASE(AM, BMN, E) \
  if (key == ((AM) | ((BMN) << 1)) && epi == (E)) return launch<BN, (AM) != 0, (BMN) != 0, (E)>(p, grid_limit, s);
#define PF_GEMM_EPIS(AM, BMN)                 \
  PF_GEMM_CASE(AM, BMN, EPI_STORE_BF16)       \
  PF_GEMM_CASE(AM, BMN, EPI_ADD_BF16)         \
  PF_GEMM_CASE(AM, BMN, EPI_ACC_F32)          \
  PF_GEMM_CASE(AM, BMN, EPI_STORE_F32)
  PF_GEMM_EPIS(0, 0)
  PF_GEMM_EPIS(0, 1)
  PF_GEMM_EPIS(1, 0)
  PF_GEMM_EPIS(1, 1)
#undef PF_GEMM_EPIS
#undef PF_GEMM_CASE
  return PF_ERR_INVALID;
}

// TMA descriptors of one problem: A logical [M, K], B logical [N, K]
int fill_problem(Problem& pr, const GemmOperand& A, const GemmOperand& B, int M, int N, int K, int block_n) {
  int rc = A.mn_major ? make_tmap(&pr.ta, A.ptr, K, M, A.ld, 64, 64) : make_tmap(&pr.ta, A.ptr, M, K, A.ld, 64, BM);
  if (rc) return rc;
  rc = B.mn_major ? make_tmap(&pr.tb, B.ptr, K, N, B.ld, 64, 64) : make_tmap(&pr.tb, B.ptr, N, K, B.ld, 64, block_n);
  if (rc) return rc;
  pr.M = M;
  pr.N = N;
  pr.tiles_m = (M + BM - 1) / BM;
  pr.tiles_n = (N + block_n - 1) / block_n;
  pr.num_tiles = pr.tiles_m * pr.tiles_n;
  pr.num_kb = (K + BK - 1) / BK;
  return PF_OK;
}

}  // namespace

int tma_desc_bf16_2d(CUtensorMap* map, const void* ptr, long long rows, long long cols, long long ld, int box_cols,
                     int box_rows) {
  return make_tmap(map, ptr, rows, cols, ld, box_cols, box_rows);
}

// fp32 row-major [rows][cols], row stride ld (elements), SWIZZLE_128B: box_cols * 4 <= 128 (TMA
// reduce-add targets)
int tma_desc_f32_2d(CUtensorMap* map, const void* ptr, long long rows, long long cols, long long ld, int box_cols,
                    int box_rows) {
  auto encode = get_encode();
  if (!encode) return PF_ERR_CUDA;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 4)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? PF_OK : PF_ERR_INVALID;
}

int tma_desc_bf16_2d_sw64(CUtensorMap* map, const void* ptr, long long rows, long long cols, long long ld,
                          int box_cols, int box_rows) {
  return make_tmap(map, ptr, rows, cols, ld, box_cols, box_rows, CU_TENSOR_MAP_SWIZZLE_64B);
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

int gemm_bf16(const GemmOperand& A, const GemmOperand& B, const GemmOut& C, int M, int N, int K, float alpha,
              int epi, int block_n, cudaStream_t stream) {
  if (M <= 0 || N <= 0 || K <= 0 || (K % 8) != 0) return PF_ERR_INVALID;
  if (block_n != 128 && block_n != 256) return PF_ERR_INVALID;
  // the epilogue moves 16-byte vectors: output rows must be 16-byte aligned
  const int esz = (epi == EPI_STORE_F32 || epi == EPI_ACC_F32) ? 4 : 2;
  if ((C.ld * esz) % 16 != 0 || reinterpret_cast<uintptr_t>(C.ptr) % 16 != 0) return PF_ERR_INVALID;
  if (epi == EPI_ACC_F32 && (C.unit_stamp == nullptr || block_n != 128)) return PF_ERR_INVALID;
  GemmParams<1> p{};
  p.nprob = 1;
  p.alpha = alpha;
  p.list_mode = 0;
  p.unit_stamp = C.unit_stamp;
  p.stamp = C.stamp;
  Problem& pr = p.prob[0];
  if (int rc = fill_problem(pr, A, B, M, N, K, block_n)) return rc;
  pr.C = C.ptr;
  pr.ldc = C.ld;
  pr.stamp_offset = C.stamp_offset;
  return block_n == 256 ? dispatch<256>(A.mn_major, B.mn_major, p, epi, pr.num_tiles, stream)
                        : dispatch<128>(A.mn_major, B.mn_major, p, epi, pr.num_tiles, stream);
}

int gemm_dw_units(const DwGemm* items, int n, int* unit_stamp, int stamp, cudaStream_t stream) {
  if (n < 0 || unit_stamp == nullptr) return PF_ERR_INVALID;
  for (int base = 0; base < n; base += kMaxDwProblems) {
    const int cnt = std::min(kMaxDwProblems, n - base);
    GemmParams<kMaxDwProblems> p{};
    p.nprob = cnt;
    p.alpha = 1.0f;
    p.list_mode = 1;
    p.unit_stamp = unit_stamp;
    p.stamp = stamp;
    long long max_units = 0;
    for (int i = 0; i < cnt; ++i) {
      const DwGemm& it = items[base + i];
      if (it.M <= 0 || it.N <= 0 || it.K <= 0 || (it.K % 8) != 0 || !it.list || !it.count || !it.C)
        return PF_ERR_INVALID;
      Problem& pr = p.prob[i];
      if (int rc = fill_problem(pr, GemmOperand{it.dy, it.ldy, true}, GemmOperand{it.x, it.ldx, true}, it.M, it.N,
                                it.K, 128))
        return rc;
      pr.C = it.C;
      pr.ldc = it.ldc;
      pr.list = it.list;
      pr.count = it.count;
      pr.stamp_offset = it.stamp_offset;
      max_units += pr.num_tiles;
    }
    if (int rc = launch<128, true, true, EPI_ACC_F32, kMaxDwProblems>(
            p, static_cast<int>(std::min<long long>(max_units, num_sms())), stream))
      return rc;
  }
  return PF_OK;
}

int gemm_bf16_units(const GemmOperand& A, const GemmOperand& B, const GemmOut& C, int M, int N, int K, float alpha,
                    const int* unit_list, const int* unit_count, int max_units, cudaStream_t stream) {
  (void)max_units;
  if (M <= 0 || N <= 0 || !A.mn_major || !B.mn_major || alpha != 1.0f) return PF_ERR_INVALID;
  DwGemm it{A.ptr, A.ld, B.ptr, B.ld, static_cast<float*>(C.ptr), C.ld, M, N, K, unit_list, unit_count,
            C.stamp_offset};
  return gemm_dw_units(&it, 1, C.unit_stamp, C.stamp, stream);
}

}  // namespace pf
