// K1 / K2 on a CTA pair: tcgen05.mma.cta_group::2, 256 x BN tiles, stream-K.
//
// Same contract as gemm.cu (C (op)= alpha * A . B^T, A K-major, B K- or
// MN-major) but each tile is computed by two CTAs of a cluster on two SMs of
// one TPC: CTA r stages rows [128 r, 128 r + 128) of A and half of B's BN rows;
// the leader (even) CTA issues the 256 x BN x 16 MMAs, which read A and B from
// both CTAs' shared memory and accumulate rows of CTA r into CTA r's TMEM. Per
// SM this halves the B traffic from L2 and shared memory relative to the
// 1-CTA 128 x BN tile, the limiter of the 1-CTA kernel (tensor pipe 57-73%).
//
// Pipelines: smem ring (each CTA's TMA signals the LEADER's full barrier with
// .cta_group::2; the leader expects both CTAs' bytes; the leader's commit
// multicasts the empty barrier to both CTAs), TMEM double buffer (leader
// commit multicasts tmem-full to both; both CTAs' epilogues arrive on the
// leader's tmem-empty barrier through shared::cluster addresses).
//
// Stream-K: when the tile count leaves the last wave of clusters mostly idle
// (the N = hidden GEMMs of a LLaMA layer: 128 tiles on 74 clusters), the full
// waves run data-parallel (one whole tile per work item) and only the tiles of
// the last, partial wave are split: their tile x k-block iterations are divided
// evenly over ALL clusters (mode 2, "DP + stream-K tail"; mode 1 splits every
// tile that way). A cluster whose range STARTS inside a tile computes that
// piece first and parks the fp32 partial in its workspace slot; the cluster
// whose range holds the tile's first k-block computes the head last, waits for
// the parked pieces of every later cluster that covers the tile, adds them and
// writes C. Only a cluster's first piece can start mid-tile, so one slot per
// cluster suffices.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "pf_device_internal.hpp"
#include "kernel_util.cuh"
#include "ptx.cuh"

namespace pf {

int tma_desc_bf16_2d(CUtensorMap* map, const void* ptr, long long rows, long long cols, long long ld, int box_cols,
                     int box_rows);
int tma_desc_bf16_2d_sw64(CUtensorMap* map, const void* ptr, long long rows, long long cols, long long ld,
                          int box_cols, int box_rows);

namespace {

#ifndef PF_STORE_NBUF
#define PF_STORE_NBUF 3
#endif
constexpr bool kStore3 = PF_STORE_NBUF == 3;
constexpr int BM2 = 256;  // rows per CTA pair
constexpr int BK = 64;
constexpr int kEpiWarps = 8;  // two warps per TMEM lane quarter, alternating 32-column chunks
constexpr int kEpiThreads = 32 * kEpiWarps;
constexpr int kThreads = 64 + kEpiThreads;

template <int BN, int EPI = EPI_STORE_BF16>
struct Cfg2 {
  // The SwiGLU epilogues give one ring stage to two epilogue buffers staged through TMA:
  // EPI_DSWIGLU gate|up of one 32-column chunk (in by TMA, overwritten by d(gate)|d(up), out by
  // TMA: 16 KB); EPI_SWIGLU gate|up|act of one chunk (out by TMA: 24 KB).
  // EPI_STORE_BF16 / EPI_ADD_BF16: two 8 KB buffers (one 128 x 32 box of C, R read in place).
  static constexpr bool TMA_EPI =
      EPI == EPI_DSWIGLU || EPI == EPI_SWIGLU || EPI == EPI_GELU || EPI == EPI_DGELU || EPI == EPI_ROPE;
  static constexpr bool TMA_PLAIN = EPI == EPI_STORE_BF16 || EPI == EPI_ADD_BF16;
  static constexpr int STAGES = TMA_EPI ? 5 : 6;
  static constexpr int A_BYTES = 128 * BK * 2;       // this CTA's half of A
  static constexpr int B_BYTES = (BN / 2) * BK * 2;  // this CTA's half of B
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int EPI_BUF =
      EPI == EPI_SWIGLU ? 3 * 8192 : ((EPI == EPI_DSWIGLU || EPI == EPI_GELU || EPI == EPI_ROPE) ? 2 * 8192 : 8192);
  // EPI_GELU and the TMA-staged EPI_STORE_BF16 cycle three buffers (one named barrier per chunk;
  // EPI_DGELU measured slower with three, profiles/r2_vit_gemm_ab.txt)
  static constexpr int EPI_NBUF = (EPI == EPI_GELU || (EPI == EPI_STORE_BF16 && kStore3)) ? 3 : 2;
  static constexpr int EPI_BYTES = (TMA_EPI || TMA_PLAIN) ? EPI_NBUF * EPI_BUF : 0;
  // EPI_DGELU column sums: [2 accumulator buffers][4 row quarters][BN] fp32
  static constexpr int CS_BYTES = EPI == EPI_DGELU ? 2 * 4 * BN * 4 : 0;
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + EPI_BYTES + CS_BYTES + 256;
};

struct alignas(64) Params2 {
  CUtensorMap ta;
  CUtensorMap tb;
  // TMA-staged epilogues, 128-row x 32-column boxes, SWIZZLE_64B:
  //   EPI_DSWIGLU  te_in = gate|up (R)         te_out = d(gate|up) (C)
  //   EPI_SWIGLU   te_in = gate|up out (C)     te_out = act (aux)
  //   EPI_GELU     te_in = pre out (C)         te_out = act (aux)
  //   EPI_DGELU    te_in = pre (R)             te_out = d(pre) (C)
  //   EPI_ADD_BF16 te_in = residual (R)        te_out = C
  //   EPI_STORE_BF16                           te_out = C
  CUtensorMap te_in;
  CUtensorMap te_out;
  int tma_epi;  // EPI_STORE_BF16 / EPI_ADD_BF16: 1 = staged through TMA (no stream-K, N % 32 == 0)
  void* C;
  long long ldc;
  int M, N, K;
  int tiles_m, tiles_n;
  int group_m;   // tile rows per raster group (B tiles are re-read once per group)
  float alpha;
  const __nv_bfloat16* R;  // EPI_ADD_BF16 residual source (defaults to C)
  long long ldr;
  __nv_bfloat16* aux;  // EPI_SWIGLU activation output
  long long ldaux;
  const __nv_bfloat16* bias;  // EPI_STORE_BF16 / EPI_ADD_BF16: + bias[col] (nullptr: none)
  float* colsum;              // EPI_DGELU: += column sums of d(pre) (the fc1 bias gradient; nullptr: none)
  const float2* rope;         // EPI_ROPE: (cos, sin) [seq][32]
  int rope_seq, rope_cols, rope_hd;
  int split_from;  // whole-tile work items: tiles [split_from, ntiles) run as two BN/2-wide halves
  int items;       // work items without stream-K: split_from + 2 * (ntiles - split_from)
  int streamk;   // 0: one tile per work item; 1/2: stream-K (2: data-parallel full waves first)
  int dp_tiles;  // stream-K: tiles [0, dp_tiles) run whole, round-robin over the clusters
  long long sk_q;  // stream-K: iterations of the split region per cluster
  float* ws;     // stream-K partials: [cluster][rank][128][BN] fp32
  int* flags;    // stream-K: [cluster][rank] == epoch once the partial is parked
  int epoch;
};

struct Seg {
  int tile, kb0, kb1;
};

// Work items of one cluster, identical for the producer, MMA and epilogue roles.
struct SegIter {
  long long next, end;  // stream-K iteration cursor
  int t;                // data-parallel tile cursor
};

__device__ __forceinline__ bool next_seg(const Params2& p, int cluster, int nclusters, int num_kb, SegIter& it,
                                         Seg& s) {
  if (!p.streamk) {
    if (it.t >= p.items) return false;
    s = Seg{it.t, 0, num_kb};
    it.t += nclusters;
    return true;
  }
  // split pieces first (a head's parked pieces are the FIRST pieces of the next clusters, so
  // they are ready when it needs them, and its fixup epilogue overlaps a whole tile's MMAs),
  // then the data-parallel tiles
  if (it.next < it.end) {
    s.tile = static_cast<int>(it.next / num_kb);
    s.kb0 = static_cast<int>(it.next - static_cast<long long>(s.tile) * num_kb);
    s.kb1 = static_cast<int>(std::min<long long>(num_kb, s.kb0 + (it.end - it.next)));
    it.next += s.kb1 - s.kb0;
    return true;
  }
  if (it.t >= p.dp_tiles) return false;
  s = Seg{it.t, 0, num_kb};
  it.t += nclusters;
  return true;
}

__device__ __forceinline__ SegIter seg_begin(const Params2& p, int cluster, int nclusters, int num_kb) {
  SegIter it{0, 0, cluster};
  if (p.streamk) {
    const long long base = static_cast<long long>(p.dp_tiles) * num_kb;
    const long long total = static_cast<long long>(p.tiles_m) * p.tiles_n * num_kb;
    it.next = std::min<long long>(total, base + static_cast<long long>(cluster) * p.sk_q);
    it.end = std::min<long long>(total, it.next + p.sk_q);
  }
  return it;
}

__device__ __forceinline__ void decode(const Params2& p, int t, int& tm, int& tn) {
  const int group_size = p.group_m * p.tiles_n;
  const int g = t / group_size;
  const int first_m = g * p.group_m;
  const int gm = min(p.tiles_m - first_m, p.group_m);
  const int local = t - g * group_size;
  tm = first_m + local % gm;
  tn = local / gm;
}

// Work item -> tile and column range. Without stream-K, the last partial wave's tiles (index >=
// split_from) are split into two BN/2-wide halves so the wave's pieces cover (nearly) every CTA pair:
// 3.46 waves of 256 x 256 tiles (the LLaMA-8B N = 4096 GEMMs) become 3 full waves + one of halves.
template <int BN>
__device__ __forceinline__ void decode_seg(const Params2& p, int item, int& tm, int& tn, int& n_begin, int& width) {
  if (item >= p.split_from) {
    const int u = item - p.split_from;
    decode(p, p.split_from + (u >> 1), tm, tn);
    n_begin = tn * BN + (u & 1) * (BN / 2);
    width = BN / 2;
  } else {
    decode(p, item, tm, tn);
    n_begin = tn * BN;
    width = BN;
  }
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int BN, bool B_MN, int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm_tcgen05_pair_kernel(const __grid_constant__ Params2 p) {
  using Cfg = Cfg2<BN, EPI>;
  constexpr int STAGES = Cfg::STAGES;
  constexpr uint32_t IDESC = idesc_bf16_f32(BM2, BN, false, B_MN);
  constexpr uint32_t IDESC_HALF = idesc_bf16_f32(BM2, BN / 2, false, B_MN);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * Cfg::A_BYTES;
  uint8_t* sE = smem + STAGES * Cfg::STAGE_BYTES;  // EPI_DSWIGLU buffers (1024-aligned)
  float* csum = reinterpret_cast<float*>(sE + Cfg::EPI_BYTES);  // EPI_DGELU column sums
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(sE + Cfg::EPI_BYTES + Cfg::CS_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* ebar = tempty_bar + 2;  // TMA-in epilogues: epilogue buffer k loaded
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ebar + 2);

  const int warp = static_cast<int>(warp_uniform(threadIdx.x >> 5));  // uniform: MMA issue stays on the uniform datapath
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1;
  const int nclusters = gridDim.x >> 1;
  const int num_kb = (p.K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 2 * kEpiThreads);
      mbar_init(&ebar[b], 1);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&p.ta);
    tma_prefetch(&p.tb);
    if (Cfg::TMA_EPI || (Cfg::TMA_PLAIN && p.tma_epi)) {
      tma_prefetch(&p.te_in);
      tma_prefetch(&p.te_out);
    }
  }
  if (warp == 1) {
    tmem_alloc_pair(tmem_slot, Cfg::TMEM_COLS);
    tmem_relinquish_pair();
  }
  tc_fence_before();
  cluster_sync_all();  // barrier inits and TMEM allocation visible to both CTAs
  tc_fence_after();
  const uint32_t tmem_base = warp_uniform(*tmem_slot);
  pdl_wait();  // setup above overlapped the preceding kernel; operands are its outputs

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------- producer (both CTAs)
      int stage = 0;
      uint32_t phase = 0;
      SegIter it = seg_begin(p, cluster, nclusters, num_kb);
      Seg sg;
      while (next_seg(p, cluster, nclusters, num_kb, it, sg)) {
        int tm, tn, nb, width;
        decode_seg<BN>(p, sg.tile, tm, tn, nb, width);
        const int m0 = tm * BM2 + static_cast<int>(rank) * 128;
        // a half-width tile loads the same boxes (expect_tx unchanged); its MMA reads the first
        // width / 2 columns of each CTA's half
        const int n0 = nb + static_cast<int>(rank) * (width / 2);
        for (int kb = sg.kb0; kb < sg.kb1; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * Cfg::STAGE_BYTES);
          uint8_t* a_dst = sA + stage * Cfg::A_BYTES;
          uint8_t* b_dst = sB + stage * Cfg::B_BYTES;
          tma_load_2d_pair(a_dst, &p.ta, &full_bar[stage], kb * BK, m0);
          if constexpr (!B_MN) {
            tma_load_2d_pair(b_dst, &p.tb, &full_bar[stage], kb * BK, n0);
          } else {
#pragma unroll
            for (int c = 0; c < (BN / 2) / 64; ++c)
              tma_load_2d_pair(b_dst + c * 8192, &p.tb, &full_bar[stage], n0 + c * 64, kb * BK);
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
    if (leader) {  // whole warp: one elected lane issues (umma_*_w)
      // ---------------------------------------------------------- MMA issuer (leader CTA)
      int stage = 0;
      uint32_t phase = 0;
      int abuf = 0;
      uint32_t aphase = 0;
      SegIter it = seg_begin(p, cluster, nclusters, num_kb);
      Seg sg;
      while (next_seg(p, cluster, nclusters, num_kb, it, sg)) {
        const uint32_t idesc = warp_uniform(sg.tile >= p.split_from ? IDESC_HALF : IDESC);
        mbar_wait(&tempty_bar[abuf], aphase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(abuf * BN);
        for (int kb = sg.kb0; kb < sg.kb1; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + stage * Cfg::A_BYTES);
          const uint32_t b_base = smem_u32(sB + stage * Cfg::B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t adesc = sdesc_sw128(a_base + k * 32, 16, 1024);
            const uint64_t bdesc = B_MN ? sdesc_sw128(b_base + k * 2048, 8192, 1024)
                                        : sdesc_sw128(b_base + k * 32, 16, 1024);
            umma_bf16_pair_w(d_tmem, adesc, bdesc, idesc, (kb != sg.kb0 || k != 0) ? 1u : 0u);
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
    const int q = warp & 3;                // TMEM lane quarter this warp may access
    const int half = (warp - 2) >> 2;      // which alternate 32-column chunks it drains
    const int row = q * 32 + static_cast<int>(lane);
    const uint32_t leader_tempty0 = mapa_shared(smem_u32(&tempty_bar[0]), 0);
    const uint32_t leader_tempty1 = mapa_shared(smem_u32(&tempty_bar[1]), 0);
    int abuf = 0;
    uint32_t aphase = 0;
    uint32_t ephase = 0;  // TMA-in epilogues: bit k = parity of epilogue buffer k's barrier
    int ec = 0;  // EPI_GELU / EPI_STORE_BF16: epilogue buffer of the next chunk (running over tiles)
    SegIter it = seg_begin(p, cluster, nclusters, num_kb);
    Seg sg;
    while (next_seg(p, cluster, nclusters, num_kb, it, sg)) {
      int tm, tn, nb, width;
      decode_seg<BN>(p, sg.tile, tm, tn, nb, width);
      // stream-K roles: a piece that starts mid-tile (kb0 > 0) parks its partial in this
      // cluster's slot; a head (kb1 < num_kb) adds the pieces parked by clusters
      // cluster+1 .. last_slot (the owner of the tile's last k-block), then writes C.
      const bool park = sg.kb0 > 0;
      const bool fixup = sg.kb0 == 0 && sg.kb1 < num_kb;
      int last_slot = cluster;
      if (fixup) {
        const long long last_it = static_cast<long long>(sg.tile) * num_kb + num_kb - 1 -
                                  static_cast<long long>(p.dp_tiles) * num_kb;
        last_slot = static_cast<int>(last_it / p.sk_q);
        if (threadIdx.x == 64) {
          for (int sl = cluster + 1; sl <= last_slot; ++sl) {
            const int* f = p.flags + sl * 2 + rank;
            while (ld_acquire(f) != p.epoch) __nanosleep(64);
          }
        }
        named_bar_sync(1, kEpiThreads);
      }
      auto ws_of = [&](int sl) { return p.ws + (static_cast<long long>(sl) * 2 + rank) * 128 * BN; };
      const long long grow = static_cast<long long>(tm) * BM2 + rank * 128 + row;
      const bool row_ok = grow < p.M;
      if constexpr (EPI == EPI_DSWIGLU) {
        // acc = d(act) for activation columns [tn*BN, tn*BN + BN) of this CTA's 128 rows. For
        // each 32-column chunk c, TMA brings gate|up (two 128 x 32 boxes at gu columns
        // (j / 128) * 256 + j % 128 and +128, SWIZZLE_64B) into buffer c & 1; every thread
        // rewrites its row's 16 columns in place with d(gate)|d(up) (same arithmetic as
        // swiglu_bwd_kernel on the bf16-rounded d(act)) and one thread stores the boxes by TMA,
        // then refills the buffer with chunk c + 2. The loads of chunks 0 and 1 are issued
        // before the accumulator is ready. No stream-K.
        const int y0 = tm * BM2 + static_cast<int>(rank) * 128;
        const bool elected = threadIdx.x == 64;
        auto gate_col = [&](int c) {
          const int j = tn * BN + c * 32;
          return ((j >> 7) << 8) + (j & 127);
        };
        auto load_chunk = [&](int c) {  // elected thread
          uint8_t* buf = sE + (c & 1) * Cfg::EPI_BUF;
          bulk_wait_read0();  // the buffer's last TMA store has read it
          mbar_arrive_expect_tx(&ebar[c & 1], Cfg::EPI_BUF);
          tma_load_2d(buf, &p.te_in, &ebar[c & 1], gate_col(c), y0);
          tma_load_2d(buf + Cfg::EPI_BUF / 2, &p.te_in, &ebar[c & 1], gate_col(c) + 128, y0);
        };
        if (elected) {
          load_chunk(0);
          load_chunk(1);
        }
        mbar_wait(&tfull_bar[abuf], aphase);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          const int k = c & 1;
          uint32_t r[16];
          tmem_ld_32x32b_x16(tmem_base + (static_cast<uint32_t>(q * 32) << 16) +
                                 static_cast<uint32_t>(abuf * BN + c * 32 + half * 16),
                             r);
          mbar_wait(&ebar[k], (ephase >> k) & 1u);
          ephase ^= 1u << k;
          tmem_ld_wait();
          uint8_t* buf = sE + k * Cfg::EPI_BUF;
#pragma unroll
          for (int s2 = 0; s2 < 2; ++s2) {
            // 16-byte chunk (2 half + s2) of this row's 64 bytes, SWIZZLE_64B: chunk ^ ((row / 2) % 4)
            const int off = row * 64 + (((2 * half + s2) ^ ((row >> 1) & 3)) << 4);
            uint4* gp = reinterpret_cast<uint4*>(buf + off);
            uint4* up = reinterpret_cast<uint4*>(buf + Cfg::EPI_BUF / 2 + off);
            const uint4 graw = *gp, uraw = *up;
            const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&graw);
            const __nv_bfloat162* u2 = reinterpret_cast<const __nv_bfloat162*>(&uraw);
            uint32_t dgw[4], duw[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float2 g = __bfloat1622float2(g2[i]);
              const float2 u = __bfloat1622float2(u2[i]);
              const float2 d = __bfloat1622float2(__floats2bfloat162_rn(p.alpha * __uint_as_float(r[8 * s2 + 2 * i]),
                                                                        p.alpha * __uint_as_float(r[8 * s2 + 2 * i + 1])));
              const float s0 = sigmoid_fast(g.x), s1 = sigmoid_fast(g.y);
              duw[i] = pack_bf16x2(d.x * (g.x * s0), d.y * (g.y * s1));
              dgw[i] = pack_bf16x2(d.x * u.x * s0 * (1.f + g.x * (1.f - s0)), d.y * u.y * s1 * (1.f + g.y * (1.f - s1)));
            }
            *gp = make_uint4(dgw[0], dgw[1], dgw[2], dgw[3]);
            *up = make_uint4(duw[0], duw[1], duw[2], duw[3]);
          }
          fence_proxy_async_smem();
          named_bar_sync(1, kEpiThreads);
          if (elected) {
            tma_store_2d(&p.te_out, buf, gate_col(c), y0);
            tma_store_2d(&p.te_out, buf + Cfg::EPI_BUF / 2, gate_col(c) + 128, y0);
            bulk_commit();
            if (c + 2 < BN / 32) load_chunk(c + 2);
          }
        }
        tc_fence_before();
        mbar_arrive_cluster(abuf ? leader_tempty1 : leader_tempty0);
        abuf ^= 1;
        if (abuf == 0) aphase ^= 1;
        continue;
      }
      if constexpr (Cfg::TMA_PLAIN) {
        if (p.tma_epi) {
          // C = bf16(alpha * acc (+ R)) staged per 32-column chunk: R (EPI_ADD_BF16) arrives by TMA
          // into buffer c & 1 (chunks 0 and 1 while the MMAs run), every thread writes its row's 16
          // columns in place, one thread stores the box by TMA and refills the buffer with R of
          // chunk c + 2 once the store has read it.
          const int y0 = tm * BM2 + static_cast<int>(rank) * 128;
          const bool elected = threadIdx.x == 64;
          auto load_r = [&](int c) {  // elected thread
            uint8_t* buf = sE + (c & 1) * Cfg::EPI_BUF;
            bulk_wait_read0();
            mbar_arrive_expect_tx(&ebar[c & 1], Cfg::EPI_BUF);
            tma_load_2d(buf, &p.te_in, &ebar[c & 1], nb + c * 32, y0);
          };
          if (EPI == EPI_ADD_BF16 && elected) {
            load_r(0);
            load_r(1);
          }
          mbar_wait(&tfull_bar[abuf], aphase);
          tc_fence_after();
          const int nchunks = width / 32;
#pragma unroll 1
          for (int c = 0; c < nchunks; ++c) {
            // EPI_STORE_BF16: three buffers over a running chunk count, as EPI_GELU; EPI_ADD_BF16: two
            const int k = (EPI == EPI_STORE_BF16 && kStore3) ? ec : c & 1;
            uint32_t r[16];
            tmem_ld_32x32b_x16(tmem_base + (static_cast<uint32_t>(q * 32) << 16) +
                                   static_cast<uint32_t>(abuf * BN + c * 32 + half * 16),
                               r);
            uint8_t* buf = sE + k * Cfg::EPI_BUF;
            if constexpr (EPI == EPI_ADD_BF16) {
              mbar_wait(&ebar[k], (ephase >> k) & 1u);
              ephase ^= 1u << k;
            } else if constexpr (!kStore3) {
              if (elected) bulk_wait_read1();
              named_bar_sync(1, kEpiThreads);
            }
            tmem_ld_wait();
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) {
              const int off = row * 64 + (((2 * half + s2) ^ ((row >> 1) & 3)) << 4);
              uint4* cp4 = reinterpret_cast<uint4*>(buf + off);
              float w[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) w[i] = p.alpha * __uint_as_float(r[8 * s2 + i]);
              if (p.bias != nullptr) {  // per-column bias (ViT linear layers); N % 32 == 0 on this path
                const uint4 braw = __ldg(reinterpret_cast<const uint4*>(p.bias + nb + c * 32 + half * 16 + 8 * s2));
                const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&braw);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  const float2 f = __bfloat1622float2(b2[i]);
                  w[2 * i] += f.x;
                  w[2 * i + 1] += f.y;
                }
              }
              if constexpr (EPI == EPI_ADD_BF16) {
                const uint4 old = *cp4;
                const __nv_bfloat162* o = reinterpret_cast<const __nv_bfloat162*>(&old);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  const float2 f = __bfloat1622float2(o[i]);
                  w[2 * i] += f.x;
                  w[2 * i + 1] += f.y;
                }
              }
              *cp4 = make_uint4(pack_bf16x2(w[0], w[1]), pack_bf16x2(w[2], w[3]), pack_bf16x2(w[4], w[5]),
                                pack_bf16x2(w[6], w[7]));
            }
            fence_proxy_async_smem();
            if (EPI == EPI_STORE_BF16 && kStore3 && elected) bulk_wait_read1();  // store c - 2 has read buffer (c + 1) % 3
            named_bar_sync(1, kEpiThreads);
            if (elected) {
              tma_store_2d(&p.te_out, buf, nb + c * 32, y0);
              bulk_commit();
              if (EPI == EPI_ADD_BF16 && c + 2 < nchunks) load_r(c + 2);
            }
            if constexpr (EPI == EPI_STORE_BF16 && kStore3) ec = ec == 2 ? 0 : ec + 1;
          }
          tc_fence_before();
          mbar_arrive_cluster(abuf ? leader_tempty1 : leader_tempty0);
          abuf ^= 1;
          if (abuf == 0) aphase ^= 1;
          continue;
        }
      }
      // EPI_ADD_BF16: the residual does not depend on the accumulator, so chunk c's 32 columns
      // are fetched while the MMAs (chunk `half`) or the previous chunk's math (c > half) run.
      uint4 rpre[4];
      auto fetch_r = [&](int c) {
        if constexpr (EPI == EPI_ADD_BF16) {
          const int gcol = nb + c * 32;
          if (!row_ok || gcol + 32 > p.N) return;
          const uint4* r4 = reinterpret_cast<const uint4*>(p.R + grow * p.ldr + gcol);
#pragma unroll
          for (int j = 0; j < 4; ++j) rpre[j] = __ldcs(r4 + j);
        }
      };
      if (EPI == EPI_ADD_BF16 && !park) fetch_r(half);
      mbar_wait(&tfull_bar[abuf], aphase);
      tc_fence_after();
      if constexpr (EPI == EPI_ROPE) {
        // qkv projection with rotate-half RoPE (head_dim 64 or 128). The tile is walked in BN / 64
        // pieces of two 128 x 32 boxes: a = columns [ca, ca + 32) of a head and its rotation
        // partner b = a + hd / 2 (hd 64: one head per piece, ca = 0; hd 128: piece c of a head,
        // ca = 32 c). The thread of (row, half) holds j in [ca + 16 half, ca + 16 half + 16) and
        // j + hd / 2, rotates them with the (cos, sin) of the row's position (q and k heads only)
        // and writes the two boxes into buffer pp & 1, stored by TMA (= GEMM then rope_fwd_kernel).
        const int y0 = tm * BM2 + static_cast<int>(rank) * 128;
        const bool elected = threadIdx.x == 64;
        const int hd = p.rope_hd;
        const float2* cs_row = p.rope + static_cast<long long>(grow % p.rope_seq) * (hd / 2);
#pragma unroll 1
        for (int pp = 0; pp < BN / 64; ++pp) {
          // columns of box a within the tile, the head's first column, j of this thread's first value
          const int head0 = hd == 64 ? pp * 64 : (pp >> 1) * 128;
          const int ca = hd == 64 ? 0 : (pp & 1) * 32;
          const int acol = head0 + ca, bcol = acol + hd / 2;
          uint32_t ra[16], rb[16];
          const uint32_t tb = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(abuf * BN);
          uint8_t* buf = sE + (pp & 1) * Cfg::EPI_BUF;
          if (pp == 0) {
            mbar_wait(&tfull_bar[abuf], aphase);
            tc_fence_after();
          }
          tmem_ld_32x32b_x16(tb + static_cast<uint32_t>(acol + half * 16), ra);
          tmem_ld_32x32b_x16(tb + static_cast<uint32_t>(bcol + half * 16), rb);
          // (cos, sin) of j in [ca + 16 half, ca + 16 half + 16) at this row's position (L1-resident)
          float2 csr[16];
          {
            const float4* c4 = reinterpret_cast<const float4*>(cs_row + ca + half * 16);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float4 v = __ldg(c4 + i);
              csr[2 * i] = make_float2(v.x, v.y);
              csr[2 * i + 1] = make_float2(v.z, v.w);
            }
          }
          if (elected) bulk_wait_read1();  // the stores of piece pp - 2 (this buffer) have read it
          named_bar_sync(1, kEpiThreads);
          tmem_ld_wait();
          const bool rot = tn * BN + head0 < p.rope_cols;
#pragma unroll
          for (int s2 = 0; s2 < 2; ++s2) {
            const int off = row * 64 + (((2 * half + s2) ^ ((row >> 1) & 3)) << 4);
            uint32_t aw[4], bw[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const __nv_bfloat162 a2 = __floats2bfloat162_rn(p.alpha * __uint_as_float(ra[8 * s2 + 2 * i]),
                                                              p.alpha * __uint_as_float(ra[8 * s2 + 2 * i + 1]));
              const __nv_bfloat162 b2 = __floats2bfloat162_rn(p.alpha * __uint_as_float(rb[8 * s2 + 2 * i]),
                                                              p.alpha * __uint_as_float(rb[8 * s2 + 2 * i + 1]));
              if (rot) {
                const float2 a = __bfloat1622float2(a2), b = __bfloat1622float2(b2);
                float oa0, ob0, oa1, ob1;
                rope_rotate(a.x, b.x, csr[8 * s2 + 2 * i], oa0, ob0);
                rope_rotate(a.y, b.y, csr[8 * s2 + 2 * i + 1], oa1, ob1);
                aw[i] = pack_bf16x2(oa0, oa1);
                bw[i] = pack_bf16x2(ob0, ob1);
              } else {
                aw[i] = *reinterpret_cast<const uint32_t*>(&a2);
                bw[i] = *reinterpret_cast<const uint32_t*>(&b2);
              }
            }
            *reinterpret_cast<uint4*>(buf + off) = make_uint4(aw[0], aw[1], aw[2], aw[3]);
            *reinterpret_cast<uint4*>(buf + 8192 + off) = make_uint4(bw[0], bw[1], bw[2], bw[3]);
          }
          fence_proxy_async_smem();
          named_bar_sync(1, kEpiThreads);
          if (elected) {
            tma_store_2d(&p.te_out, buf, tn * BN + acol, y0);
            tma_store_2d(&p.te_out, buf + 8192, tn * BN + bcol, y0);
            bulk_commit();
          }
        }
        tc_fence_before();
        mbar_arrive_cluster(abuf ? leader_tempty1 : leader_tempty0);
        abuf ^= 1;
        if (abuf == 0) aphase ^= 1;
        continue;
      }
      if constexpr (EPI == EPI_GELU || EPI == EPI_DGELU) {
        // ViT MLP, per 32-column chunk staged in buffer c & 1 (128 x 32 SWIZZLE_64B boxes):
        //   EPI_GELU:  pre = bf16(alpha acc + bias), act = gelu(pre); both boxes stored by TMA
        //              (= GEMM with bias followed by gelu_fwd_kernel, bit for bit)
        //   EPI_DGELU: pre arrives by TMA (chunks 0 and 1 while the MMAs run), is overwritten in
        //              place by d(pre) = bf16(alpha acc) * gelu'(pre), stored by TMA, and the buffer
        //              is refilled with chunk c + 2 (= GEMM then gelu_bwd_kernel, bit for bit)
        // EPI_GELU cycles three buffers: chunk c may be written once the store of chunk c - 3 has read
        // its buffer, which the elected thread checks (wait_group.read 1) before the previous chunk's
        // barrier, so each chunk needs one CTA-wide barrier instead of two.
        const int y0 = tm * BM2 + static_cast<int>(rank) * 128;
        const bool elected = threadIdx.x == 64;
        auto load_pre = [&](int c) {  // EPI_DGELU, elected thread
          uint8_t* buf = sE + (c & 1) * Cfg::EPI_BUF;
          bulk_wait_read0();
          mbar_arrive_expect_tx(&ebar[c & 1], Cfg::EPI_BUF);
          tma_load_2d(buf, &p.te_in, &ebar[c & 1], tn * BN + c * 32, y0);
        };
        if (EPI == EPI_DGELU && elected) {
          load_pre(0);
          load_pre(1);
        }
        mbar_wait(&tfull_bar[abuf], aphase);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          // EPI_GELU: three buffers over a running chunk count (tiles of 8 chunks); EPI_DGELU: two
          const int k = EPI == EPI_GELU ? ec : c & 1;
          uint32_t r[16];
          tmem_ld_32x32b_x16(tmem_base + (static_cast<uint32_t>(q * 32) << 16) +
                                 static_cast<uint32_t>(abuf * BN + c * 32 + half * 16),
                             r);
          uint8_t* buf = sE + k * Cfg::EPI_BUF;
          if constexpr (EPI == EPI_DGELU) {
            mbar_wait(&ebar[k], (ephase >> k) & 1u);
            ephase ^= 1u << k;
          }
          tmem_ld_wait();
#pragma unroll
          for (int s2 = 0; s2 < 2; ++s2) {
            const int off = row * 64 + (((2 * half + s2) ^ ((row >> 1) & 3)) << 4);
            uint4* pp = reinterpret_cast<uint4*>(buf + off);
            if constexpr (EPI == EPI_GELU) {
              float w[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) w[i] = p.alpha * __uint_as_float(r[8 * s2 + i]);
              if (p.bias != nullptr) {
                const uint4 braw =
                    __ldg(reinterpret_cast<const uint4*>(p.bias + tn * BN + c * 32 + half * 16 + 8 * s2));
                const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&braw);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  const float2 f = __bfloat1622float2(b2[i]);
                  w[2 * i] += f.x;
                  w[2 * i + 1] += f.y;
                }
              }
              uint32_t pw[4], aw[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const __nv_bfloat162 pb = __floats2bfloat162_rn(w[2 * i], w[2 * i + 1]);
                const float2 pf = __bfloat1622float2(pb);
                pw[i] = *reinterpret_cast<const uint32_t*>(&pb);
                const float2 g = gelu_erf2(pf);
                aw[i] = pack_bf16x2(g.x, g.y);
              }
              *pp = make_uint4(pw[0], pw[1], pw[2], pw[3]);
              *reinterpret_cast<uint4*>(buf + 8192 + off) = make_uint4(aw[0], aw[1], aw[2], aw[3]);
            } else {
              const uint4 praw = *pp;
              const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&praw);
              uint32_t dw[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float2 pf = __bfloat1622float2(p2[i]);
                const float2 d = __bfloat1622float2(__floats2bfloat162_rn(p.alpha * __uint_as_float(r[8 * s2 + 2 * i]),
                                                                          p.alpha * __uint_as_float(r[8 * s2 + 2 * i + 1])));
                const float2 gd = mul2(d, gelu_erf_grad2(pf));
                const __nv_bfloat162 o = __floats2bfloat162_rn(gd.x, gd.y);
                dw[i] = *reinterpret_cast<const uint32_t*>(&o);
                const float2 of = __bfloat1622float2(o);  // the stored (bf16) d(pre) feeds the bias gradient
                r[8 * s2 + 2 * i] = __float_as_uint(of.x);
                r[8 * s2 + 2 * i + 1] = __float_as_uint(of.y);
              }
              *pp = make_uint4(dw[0], dw[1], dw[2], dw[3]);
            }
          }
          fence_proxy_async_smem();
          if (EPI == EPI_GELU && elected) bulk_wait_read1();  // store c - 2 has read buffer (c + 1) % 3
          named_bar_sync(1, kEpiThreads);
          if (EPI == EPI_DGELU && p.colsum != nullptr) {
            // column sums over this warp's 32 rows of its 16 columns, from registers (r holds the
            // bf16-rounded d(pre)): a butterfly reduce-scatter, 16 shuffles; lane l ends with the sum
            // of column (l >> 1) & 15 (lanes l, l ^ 1 agree). Rows past M are TMA zero-fill: 0.
            float v[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
            // round (W values move, lane bit B, partner lane ^ 2^B): keep the half selected by bit B
#define PF_CS_ROUND(W, B)                                              \
  {                                                                    \
    const bool up = (lane >> (B)) & 1u;                                \
    _Pragma("unroll") for (int j = 0; j < (W); ++j) {                  \
      const float send = up ? v[j] : v[j + (W)];                       \
      const float keep = up ? v[j + (W)] : v[j];                       \
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, 1 << (B));      \
    }                                                                  \
  }
            PF_CS_ROUND(8, 4)
            PF_CS_ROUND(4, 3)
            PF_CS_ROUND(2, 2)
            PF_CS_ROUND(1, 1)
#undef PF_CS_ROUND
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
            if ((lane & 1u) == 0)
              csum[(abuf * 4 + q) * BN + c * 32 + half * 16 + static_cast<int>((lane >> 1) & 15u)] = v[0];
          }
          if (elected) {
            if constexpr (EPI == EPI_GELU) {
              tma_store_2d(&p.te_in, buf, tn * BN + c * 32, y0);
              tma_store_2d(&p.te_out, buf + 8192, tn * BN + c * 32, y0);
              bulk_commit();
            } else {
              tma_store_2d(&p.te_out, buf, tn * BN + c * 32, y0);
              bulk_commit();
              if (c + 2 < BN / 32) load_pre(c + 2);
            }
          }
          if constexpr (EPI == EPI_GELU) ec = ec == 2 ? 0 : ec + 1;
        }
        if (EPI == EPI_DGELU && p.colsum != nullptr) {
          // one atomic per column per CTA and tile (csum is double-buffered by accumulator buffer:
          // the next tile's writes go to the other half, and the one after follows 8 named barriers)
          named_bar_sync(1, kEpiThreads);
          for (int cc = threadIdx.x - 64; cc < BN; cc += kEpiThreads) {
            const float* cs = csum + abuf * 4 * BN + cc;
            const int gcol = tn * BN + cc;
            if (gcol < p.N) atomicAdd(p.colsum + gcol, cs[0] + cs[BN] + cs[2 * BN] + cs[3 * BN]);
          }
        }
        tc_fence_before();
        mbar_arrive_cluster(abuf ? leader_tempty1 : leader_tempty0);
        abuf ^= 1;
        if (abuf == 0) aphase ^= 1;
        continue;
      }
      if constexpr (EPI == EPI_SWIGLU) {
        // columns [0, BN/2) of the tile are gate j, [BN/2, BN) up j (host: N % BN == 0, no stream-K);
        // the activation uses the bf16-rounded gate/up exactly as swiglu_fwd_kernel does. Each
        // 32-column chunk c of gate, up and act is written to buffer c & 1 (three 128 x 32
        // SWIZZLE_64B boxes) and stored by TMA, so HBM sees whole lines.
        const int y0 = tm * BM2 + static_cast<int>(rank) * 128;
        const bool elected = threadIdx.x == 64;
#pragma unroll 1
        for (int c = 0; c < BN / 64; ++c) {
          uint32_t rg[16], ru[16];
          const uint32_t tbase = tmem_base + (static_cast<uint32_t>(q * 32) << 16) +
                                 static_cast<uint32_t>(abuf * BN + c * 32 + half * 16);
          tmem_ld_32x32b_x16(tbase, rg);
          tmem_ld_32x32b_x16(tbase + BN / 2, ru);
          uint8_t* buf = sE + (c & 1) * Cfg::EPI_BUF;
          if (elected) bulk_wait_read1();  // the store of chunk c - 2 (this buffer) has read it
          named_bar_sync(1, kEpiThreads);
          tmem_ld_wait();
#pragma unroll
          for (int s2 = 0; s2 < 2; ++s2) {
            const int off = row * 64 + (((2 * half + s2) ^ ((row >> 1) & 3)) << 4);
            uint32_t gw[4], uw[4], aw[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const __nv_bfloat162 g2 = __floats2bfloat162_rn(p.alpha * __uint_as_float(rg[8 * s2 + 2 * i]),
                                                              p.alpha * __uint_as_float(rg[8 * s2 + 2 * i + 1]));
              const __nv_bfloat162 u2 = __floats2bfloat162_rn(p.alpha * __uint_as_float(ru[8 * s2 + 2 * i]),
                                                              p.alpha * __uint_as_float(ru[8 * s2 + 2 * i + 1]));
              const float2 g = __bfloat1622float2(g2);
              const float2 u = __bfloat1622float2(u2);
              gw[i] = *reinterpret_cast<const uint32_t*>(&g2);
              uw[i] = *reinterpret_cast<const uint32_t*>(&u2);
              aw[i] = pack_bf16x2(g.x * sigmoid_fast(g.x) * u.x, g.y * sigmoid_fast(g.y) * u.y);
            }
            *reinterpret_cast<uint4*>(buf + off) = make_uint4(gw[0], gw[1], gw[2], gw[3]);
            *reinterpret_cast<uint4*>(buf + 8192 + off) = make_uint4(uw[0], uw[1], uw[2], uw[3]);
            *reinterpret_cast<uint4*>(buf + 16384 + off) = make_uint4(aw[0], aw[1], aw[2], aw[3]);
          }
          fence_proxy_async_smem();
          named_bar_sync(1, kEpiThreads);
          if (elected) {
            tma_store_2d(&p.te_in, buf, tn * BN + c * 32, y0);
            tma_store_2d(&p.te_in, buf + 8192, tn * BN + BN / 2 + c * 32, y0);
            tma_store_2d(&p.te_out, buf + 16384, tn * (BN / 2) + c * 32, y0);
            bulk_commit();
          }
        }
        tc_fence_before();
        mbar_arrive_cluster(abuf ? leader_tempty1 : leader_tempty0);
        abuf ^= 1;
        if (abuf == 0) aphase ^= 1;
        continue;
      }
#pragma unroll 1
      for (int c = half; c < width / 32; c += 2) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) +
                               static_cast<uint32_t>(abuf * BN + c * 32),
                           r);
        const uint4 rcur[4] = {rpre[0], rpre[1], rpre[2], rpre[3]};
        if (EPI == EPI_ADD_BF16 && !park && c + 2 < width / 32) fetch_r(c + 2);
        tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
        if (park) {  // raw fp32 partial, row-major within the slot
          float4* w = reinterpret_cast<float4*>(ws_of(cluster) + static_cast<long long>(row) * BN + c * 32);
#pragma unroll
          for (int j = 0; j < 8; ++j) w[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          continue;
        }
        if (fixup) {
          for (int sl = cluster + 1; sl <= last_slot; ++sl) {
            const float4* w = reinterpret_cast<const float4*>(ws_of(sl) + static_cast<long long>(row) * BN + c * 32);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float4 o = __ldcg(w + j);
              v[4 * j] += o.x;
              v[4 * j + 1] += o.y;
              v[4 * j + 2] += o.z;
              v[4 * j + 3] += o.w;
            }
          }
        }
        const int gcol = nb + c * 32;
        if (!row_ok || gcol >= p.N) continue;
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] *= p.alpha;
        const bool full = gcol + 32 <= p.N;
        if (p.bias != nullptr) {  // per-column bias (ViT linear layers), same for every row
          if (full) {
            const uint4* b4 = reinterpret_cast<const uint4*>(p.bias + gcol);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint4 braw = __ldg(b4 + j);
              const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&braw);
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float2 f = __bfloat1622float2(b2[i]);
                v[8 * j + 2 * i] += f.x;
                v[8 * j + 2 * i + 1] += f.y;
              }
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (gcol + i < p.N) v[i] += __bfloat162float(p.bias[gcol + i]);
          }
        }
        if constexpr (EPI == EPI_STORE_BF16 || EPI == EPI_ADD_BF16) {
          __nv_bfloat16* cp = reinterpret_cast<__nv_bfloat16*>(p.C) + grow * p.ldc + gcol;
          const __nv_bfloat16* rp = p.R + grow * p.ldr + gcol;
          if (full) {
            uint4* c4 = reinterpret_cast<uint4*>(cp);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              float w[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) w[i] = v[j * 8 + i];
              if constexpr (EPI == EPI_ADD_BF16) {
                const uint4 old = rcur[j];
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
              if (gcol + i < p.N) {
                float w = v[i];
                if constexpr (EPI == EPI_ADD_BF16) w += __bfloat162float(rp[i]);
                cp[i] = __float2bfloat16_rn(w);
              }
            }
          }
        } else {
          float* cp = reinterpret_cast<float*>(p.C) + grow * p.ldc + gcol;
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (gcol + i < p.N) cp[i] = v[i];
        }
      }
      tc_fence_before();
      mbar_arrive_cluster(abuf ? leader_tempty1 : leader_tempty0);
      if (park) {  // publish the partial once all 128 epilogue threads wrote their rows
        named_bar_sync(1, kEpiThreads);
        if (threadIdx.x == 64) {
          __threadfence();
          st_release(p.flags + cluster * 2 + rank, p.epoch);
        }
      }
      abuf ^= 1;
      if (abuf == 0) aphase ^= 1;
    }
    if ((Cfg::TMA_EPI || Cfg::TMA_PLAIN) && threadIdx.x == 64) bulk_wait0();  // the last TMA stores have landed
  }

  tc_fence_before();
  cluster_sync_all();  // both CTAs done with TMEM and with each other's barriers
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, Cfg::TMEM_COLS);
  }
}

// Co-resident CTA pairs for this kernel (stream-K waits across clusters, so its
// grid must never exceed what the GPU can hold at once).
template <int BN, bool B_MN, int EPI>
int max_active_clusters() {
  using Cfg = Cfg2<BN, EPI>;
  static int n = -1;
  if (n < 0) {
    auto kern = gemm_tcgen05_pair_kernel<BN, B_MN, EPI>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * (num_sms() / 2));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
    cudaLaunchAttribute attr{};
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = 2;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int c = 0;
    if (cudaOccupancyMaxActiveClusters(&c, kern, &cfg) != cudaSuccess || c <= 0) {
      cudaGetLastError();
      c = num_sms() / 2;
    }
    n = std::min(c, num_sms() / 2);
  }
  return n;
}

template <int BN, bool B_MN, int EPI>
int launch2(Params2 p, int clusters, cudaStream_t stream) {
  using Cfg = Cfg2<BN, EPI>;
  auto kern = gemm_tcgen05_pair_kernel<BN, B_MN, EPI>;
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES) != cudaSuccess)
      return PF_ERR_CUDA;
    attr_set = true;
  }
  const int active = max_active_clusters<BN, B_MN, EPI>();
  if (p.streamk && clusters > active) return PF_ERR_INVALID;  // ranges were cut for `clusters`
  clusters = std::min(clusters, active);
  if (clusters <= 0) return PF_OK;
  launch_k(kern, dim3(2 * clusters), dim3(kThreads), Cfg::SMEM_BYTES, stream, p);
  count_launch();
  return cudaPeekAtLastError() == cudaSuccess ? PF_OK : PF_ERR_CUDA;
}

// Stream-K workspace (per device process; kernels on one stream use it in order).
struct StreamKState {
  float* ws = nullptr;
  int* flags = nullptr;
  int slots = 0;
  int epoch = 0;
};

StreamKState& sk_state() {
  static StreamKState st;
  return st;
}

int& streamk_mode_ref() {
  // 0 off (default), 1 every tile split, 2 data-parallel full waves + split last wave, -1 auto
  // (mode 2 where the last wave would leave > 8% of the CTA pairs idle). Both split forms
  // measured slower than whole tiles on B200 for every LLaMA shape, including the 1.73-wave
  // N = 2048 GEMMs they target (profiles/r1_gemm_bench_streamk.txt).
  static int mode = [] {
    const char* e = std::getenv("PF_GEMM_STREAMK");
    return e ? std::atoi(e) : 0;
  }();
  return mode;
}
int streamk_mode() { return streamk_mode_ref(); }

// PF_GEMM_TAIL_SPLIT=0: the last partial wave runs whole tiles too (A/B)
bool tail_split_on() {
  const char* e = std::getenv("PF_GEMM_TAIL_SPLIT");
  return !(e && e[0] == '0');
}

// K1/K2 plain epilogues through shared memory + TMA stores (PF_GEMM_TMA_EPI=0: row-per-thread stores)
bool tma_plain_epi() {
  static const bool on = [] {
    const char* e = std::getenv("PF_GEMM_TMA_EPI");
    return !(e && e[0] == '0');
  }();
  return on;
}

}  // namespace

void gemm_set_streamk(int mode) { streamk_mode_ref() = mode; }

// Raster group height in 256-row tiles: consecutive work items walk G tile rows down one
// tile column before moving right, so each B column block is fetched once per group and
// the G row blocks of A stay hot in L2. Chosen per shape from B200 measurements
// (profiles/r1_gemm_group_m.txt): wide forward GEMMs with short K keep all of A resident
// (G = 16: B streamed once; lm head 1391 -> 1576 TF/s); dX GEMMs (B read MN-major) and
// long-K shapes prefer short groups (gate|up dX 1082 -> 1270 TF/s at G = 4).
// PF_GEMM_GROUP_M overrides.
int group_m_for(int tiles_m, int tiles_n, int K, bool b_mn) {
  static const int forced = [] {
    const char* e = std::getenv("PF_GEMM_GROUP_M");
    return e ? std::atoi(e) : 0;
  }();
  if (forced > 0) return forced;
  // Wide forward GEMMs with at most 16 tile rows take them all in one group at any K, so each weight
  // column block is read from DRAM once (the 4096-row A stays in L2): the LLaMA-8B gate|up read its
  // 235 MB weight twice at G = 8; C3 +0.6-0.8% tok/s (profiles/r2_gemm_fullm.md). PF_GEMM_FULLM=0: G = 8.
  static const bool fullm = [] {
    const char* e = std::getenv("PF_GEMM_FULLM");
    return !(e && e[0] == '0');
  }();
  if (!b_mn && tiles_n >= 48 && fullm && tiles_m <= 16) return tiles_m;
  if (!b_mn && tiles_n >= 48) return K <= 2048 ? std::min(tiles_m, 16) : 8;
  return K >= 32768 ? 8 : 4;
}

int gemm_bf16_pair(const GemmOperand& A, const GemmOperand& B, const GemmOut& C, int M, int N, int K, float alpha,
                   int epi, cudaStream_t stream) {
  constexpr int BN = 256;
  if (M <= 0 || N <= 0 || K <= 0 || (K % 8) != 0 || A.mn_major) return PF_ERR_INVALID;
  // the epilogues move 16-byte vectors: output and residual rows must be 16-byte aligned
  const int esz = epi == EPI_STORE_F32 ? 4 : 2;
  if ((C.ld * esz) % 16 != 0 || reinterpret_cast<uintptr_t>(C.ptr) % 16 != 0 ||
      (C.residual && ((C.ldr * 2) % 16 != 0 || reinterpret_cast<uintptr_t>(C.residual) % 16 != 0)))
    return PF_ERR_INVALID;
  Params2 p{};
  int rc = tma_desc_bf16_2d(&p.ta, A.ptr, M, K, A.ld, 64, 128);
  if (rc) return rc;
  rc = B.mn_major ? tma_desc_bf16_2d(&p.tb, B.ptr, K, N, B.ld, 64, 64)
                  : tma_desc_bf16_2d(&p.tb, B.ptr, N, K, B.ld, 64, BN / 2);
  if (rc) return rc;
  p.C = C.ptr;
  p.ldc = C.ld;
  p.R = static_cast<const __nv_bfloat16*>(C.residual ? C.residual : C.ptr);
  p.ldr = C.residual ? C.ldr : C.ld;
  p.aux = static_cast<__nv_bfloat16*>(C.aux);
  p.ldaux = C.ldaux;
  p.bias = static_cast<const __nv_bfloat16*>(C.bias);
  if (p.bias && epi != EPI_STORE_BF16 && epi != EPI_ADD_BF16 && epi != EPI_GELU) return PF_ERR_INVALID;
  if (epi == EPI_ROPE) {  // qkv [M][N] out by TMA, q/k heads of 64 or 128 columns rotated
    if (N % BN != 0 || B.mn_major || !C.rope || C.rope_seq <= 0 || (C.rope_hd != 64 && C.rope_hd != 128) ||
        C.rope_cols % C.rope_hd != 0)
      return PF_ERR_INVALID;
    p.rope_hd = C.rope_hd;
    if ((rc = tma_desc_bf16_2d_sw64(&p.te_out, C.ptr, M, N, C.ld, 32, 128))) return rc;
    p.rope = static_cast<const float2*>(C.rope);
    p.rope_seq = C.rope_seq;
    p.rope_cols = C.rope_cols;
  }
  if (epi == EPI_GELU) {  // pre [M][N] and act [M][N] out by TMA
    if (N % 32 != 0 || B.mn_major || !C.aux) return PF_ERR_INVALID;
    if ((rc = tma_desc_bf16_2d_sw64(&p.te_in, C.ptr, M, N, C.ld, 32, 128))) return rc;
    if ((rc = tma_desc_bf16_2d_sw64(&p.te_out, C.aux, M, N, C.ldaux, 32, 128))) return rc;
  }
  p.colsum = C.colsum;
  if (C.colsum && epi != EPI_DGELU) return PF_ERR_INVALID;
  if (epi == EPI_DGELU) {  // pre [M][N] in, d(pre) [M][N] out by TMA (may be the same buffer)
    if (N % 32 != 0 || !B.mn_major || !C.residual || C.bias) return PF_ERR_INVALID;
    if ((rc = tma_desc_bf16_2d_sw64(&p.te_in, C.residual, M, N, C.ldr, 32, 128))) return rc;
    if ((rc = tma_desc_bf16_2d_sw64(&p.te_out, C.ptr, M, N, C.ld, 32, 128))) return rc;
  }
  if (epi == EPI_SWIGLU) {
    if (N % BN != 0 || B.mn_major || !C.aux) return PF_ERR_INVALID;
    // gate|up [M][N] and act [M][N/2] out by TMA, 32-column x 128-row boxes
    if ((rc = tma_desc_bf16_2d_sw64(&p.te_in, C.ptr, M, N, C.ld, 32, 128))) return rc;
    if ((rc = tma_desc_bf16_2d_sw64(&p.te_out, C.aux, M, N / 2, C.ldaux, 32, 128))) return rc;
  }
  if (epi == EPI_DSWIGLU) {
    if (N % 128 != 0 || !B.mn_major || !C.residual) return PF_ERR_INVALID;
    // gate|up in and d(gate|up) out by TMA: [M][2N] bf16, 32-column x 128-row boxes
    if ((rc = tma_desc_bf16_2d_sw64(&p.te_in, C.residual, M, 2LL * N, C.ldr, 32, 128))) return rc;
    if ((rc = tma_desc_bf16_2d_sw64(&p.te_out, C.ptr, M, 2LL * N, C.ld, 32, 128))) return rc;
  }
  p.M = M;
  p.N = N;
  p.K = K;
  p.tiles_m = (M + BM2 - 1) / BM2;
  p.tiles_n = (N + BN - 1) / BN;
  p.group_m = std::max(1, group_m_for(p.tiles_m, p.tiles_n, K, B.mn_major));
  p.alpha = alpha;
  const int ntiles = p.tiles_m * p.tiles_n;
  const int max_clusters = num_sms() / 2;
  int clusters = std::min(ntiles, max_clusters);
  // stream-K when the data-parallel last wave would leave > 8% of the clusters idle
  const int num_kb = (K + BK - 1) / BK;
  const int waves = (ntiles + max_clusters - 1) / max_clusters;
  const double eff = static_cast<double>(ntiles) / (static_cast<double>(waves) * max_clusters);
  const int mode = streamk_mode();
  const int active = std::min(max_clusters, max_active_clusters<BN, false, EPI_STORE_BF16>());
  const bool sk = epi != EPI_SWIGLU && epi != EPI_DSWIGLU && epi != EPI_GELU && epi != EPI_DGELU && epi != EPI_ROPE &&
                  (ntiles > active || mode == 1) && num_kb >= 8 &&
                  (mode == 1 || mode == 2 || (mode < 0 && eff < 0.92));
  if (sk) {
    StreamKState& st = sk_state();
    clusters = active;
    p.dp_tiles = mode == 1 ? 0 : (ntiles / clusters) * clusters;
    const long long split = static_cast<long long>(ntiles - p.dp_tiles) * num_kb;
    p.sk_q = (split + clusters - 1) / clusters;
    if (st.slots < clusters + 1) {
      if (st.ws) cudaFree(st.ws);
      if (st.flags) cudaFree(st.flags);
      if (cudaMalloc(&st.ws, static_cast<size_t>(clusters + 1) * 2 * 128 * BN * sizeof(float)) != cudaSuccess ||
          cudaMalloc(&st.flags, static_cast<size_t>(clusters + 1) * 2 * sizeof(int)) != cudaSuccess)
        return PF_ERR_CUDA;
      cudaMemset(st.flags, 0, static_cast<size_t>(clusters + 1) * 2 * sizeof(int));
      st.slots = clusters + 1;
    }
    p.streamk = mode == 1 ? 1 : 2;
    p.ws = st.ws;
    p.flags = st.flags;
    p.epoch = ++st.epoch;
  }
  if ((epi == EPI_STORE_BF16 || epi == EPI_ADD_BF16) && !p.streamk && N % 32 == 0 && tma_plain_epi()) {
    // TMA needs 16-byte aligned bases and row strides; otherwise the row-per-thread epilogue runs
    p.tma_epi = tma_desc_bf16_2d_sw64(&p.te_out, C.ptr, M, N, C.ld, 32, 128) == PF_OK &&
                (epi != EPI_ADD_BF16 || tma_desc_bf16_2d_sw64(&p.te_in, p.R, M, N, p.ldr, 32, 128) == PF_OK);
  }
  // whole tiles, except a last partial wave of at most half the CTA pairs, which runs as half-width
  // tiles (plain TMA-staged epilogues only; PF_GEMM_TAIL_SPLIT=0 turns it off)
  p.split_from = ntiles;
  p.items = ntiles;
  if (!p.streamk && p.tma_epi && tail_split_on() && ntiles > clusters) {
    const int rem = ntiles % clusters;
    if (rem > 0 && 2 * rem <= clusters) {
      p.split_from = ntiles - rem;
      p.items = ntiles + rem;
    }
  }
  const bool bmn = B.mn_major;
  switch (epi) {
    case EPI_STORE_BF16:
      return bmn ? launch2<BN, true, EPI_STORE_BF16>(p, clusters, stream)
                 : launch2<BN, false, EPI_STORE_BF16>(p, clusters, stream);
    case EPI_ADD_BF16:
      return bmn ? launch2<BN, true, EPI_ADD_BF16>(p, clusters, stream)
                 : launch2<BN, false, EPI_ADD_BF16>(p, clusters, stream);
    case EPI_STORE_F32:
      return bmn ? launch2<BN, true, EPI_STORE_F32>(p, clusters, stream)
                 : launch2<BN, false, EPI_STORE_F32>(p, clusters, stream);
    case EPI_SWIGLU:
      return launch2<BN, false, EPI_SWIGLU>(p, clusters, stream);
    case EPI_DSWIGLU:
      return launch2<BN, true, EPI_DSWIGLU>(p, clusters, stream);
    case EPI_GELU:
      return launch2<BN, false, EPI_GELU>(p, clusters, stream);
    case EPI_ROPE:
      return launch2<BN, false, EPI_ROPE>(p, clusters, stream);
    case EPI_DGELU:
      return launch2<BN, true, EPI_DGELU>(p, clusters, stream);
    default: return PF_ERR_INVALID;
  }
}

}  // namespace pf
