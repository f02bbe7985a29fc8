// K7 attention: causal (LLaMA) or bidirectional multi-head attention with native GQA, hand-written
// for sm_100a. Replaces the library fused attention the stage used before (the reference has no
// attention at all: its cost sits inside the forward / backward_act stand-ins,
// proj/src/timing.cpp:21-23, the part of the backward freezing can never shrink).
//
// Layout (stage.cpp): qkv [T, (nh + 2 nkv) hd] bf16 after RoPE, T = B * S tokens, a head's 128-row
// tile of q / k / v is read straight out of it by TMA (box 64 x 128, SWIZZLE_128B; a tile is hd/64
// such 16 KB regions). S % 128 == 0, hd in {64, 128}.
//
// Forward (flash_fwd_kernel, one CTA per (sequence, head, 128-query block), heaviest causal blocks
// first; 6 warps):
//   warp 0      TMA: Q once, then K_j and V_j into a ring of 128-row tiles
//   warp 1      TMEM allocation + the MMA issuer (one thread):
//                 S_j = Q K_j^T   tcgen05.mma, A and B from shared memory -> TMEM (two S buffers)
//                 O  += P_j V_j   A = P_j from TMEM (bf16, written over S_j), B = V_j -> TMEM O
//               S_{j+1} is issued before waiting for P_j, so the tensor pipe computes the next
//               scores while the softmax warps exponentiate the current ones.
//   warps 2-5   softmax, one thread per query row: tcgen05.ld of the S row, row max, lazy rescale of
//               O in TMEM only when the max grows by more than 2^8 (FA4-style), P = 2^(s - m) as
//               bf16 back into TMEM; epilogue O / l -> bf16 [T, nh*hd], LSE (log2 domain) [B, nh, S].
//
// Backward (flash_bwd_kernel, one CTA per (sequence, kv head, 128-key block): it loops over the
// query blocks the keys see and, inside, the rep = nh / nkv query heads of the group, so K_j / V_j
// stay in shared memory and dK / dV accumulate in TMEM; query-block-major, the CTAs of different key
// blocks that run in lockstep reduce into different dQ rows at any time):
//   S^T  = K_j Q_i^T, dP^T = V_j dO_i^T                       (TMEM, lane = key row)
//   P^T  = 2^(S^T * c - LSE_i), dS^T = P^T (dP^T - D_i)      (softmax warps; bf16 into TMEM over
//                                                              S^T / dP^T and dS^T into shared memory)
//   dV  += P^T dO_i,  dK += dS^T Q_i                          (A from TMEM)
//   dQ_i = dS K_j                                             (A = dS^T in shared memory read MN-major)
// dQ_i is drained from TMEM by the softmax warps into an fp32 accumulator (red.global.add.v4.f32);
// flash_bwd_dq_kernel then scales it, applies the RoPE backward and writes bf16 dq into the packed
// dqkv. dK (scaled, RoPE backward) and dV are written by the CTA that owns the key block, in place
// over qkv's k / v columns of that block (no other CTA reads them). flash_bwd_pre_kernel computes
// D = rowsum(dO * O) and zeroes the dQ accumulator.
// The same shared-memory tile serves as a K-major operand (rows = M/N, columns = K) and as an
// MN-major one (rows = K): SWIZZLE_128B 64-column regions are both layouts' canonical form.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "kernel_util.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

namespace pf {

int tma_desc_bf16_2d(CUtensorMap* map, const void* ptr, long long rows, long long cols, long long ld, int box_cols,
                     int box_rows);
int tma_desc_f32_2d(CUtensorMap* map, const void* ptr, long long rows, long long cols, long long ld, int box_cols,
                    int box_rows);

namespace {

// Optional cycle accounting of the first CTA's roles (PF_ATTN_PROF=1; tools/attn_bench.py --prof)
__device__ unsigned long long g_attn_prof[32];
struct ProfClock {
  bool on;
  __device__ __forceinline__ long long now() const { return on ? clock64() : 0; }
  __device__ __forceinline__ void add(int slot, long long t0) const {
    if (on) g_attn_prof[slot] += static_cast<unsigned long long>(clock64() - t0);
  }
};

constexpr float kRescaleLog2 = 8.0f;  // lazy O rescale threshold: unnormalised P stays <= 2^8
constexpr int kSoftWarps = 16;        // softmax warps: 4 per TMEM lane quarter, one 32-column slice each
constexpr int kSoftThreads = 32 * kSoftWarps;
constexpr int kAttnThreads = 64 + kSoftThreads;
constexpr int kFwd2Threads = 64 + 512;  // two-tile forward: TMA, MMA, 8 softmax warps per tile
constexpr int kDrainWarps = 4;  // backward: one dQ-drain warp per TMEM lane quarter
constexpr int kBwdThreads = kAttnThreads + 32 * kDrainWarps;

struct FwdParams {
  CUtensorMap tqkv;  // qkv [T, W], box {64, 128}
  __nv_bfloat16* out;
  long long ldo;
  float* lse;  // [B, nh, S]: m + log2(l) of the log2-scaled scores
  int B, S, nh, nkv, rep, nqb, causal, prof;
  float scale_log2;
};

struct BwdParams {
  CUtensorMap tqkv;  // qkv [T, W], box {64, 128}
  CUtensorMap tdo;   // dO [T, nh*hd], box {64, 128}
  CUtensorMap tdq;   // dQ accumulator fp32 [T, nh*hd], box {32, 32}, SWIZZLE_128B (TMA reduce-add)
  const float* lse;  // [B, nh, S]
  const float* D;    // [B, nh, S]
  float* dq_acc;     // [T, nh*hd] fp32
  __nv_bfloat16* dqkv;
  long long ldq;  // row stride of qkv / dqkv (W)
  const float2* rope;  // (cos, sin) [S][hd/2] or null
  int B, S, nh, nkv, rep, nqb, causal, prof;
  float scale_log2, scale;
};

template <int HD>
struct AttnCfg {
  static constexpr int TILE = 128 * HD * 2;  // one 128-row tile, HD/64 regions of 16 KB
  static constexpr int FWD_STAGES = HD == 128 ? 4 : 6;
  static constexpr int FWD_SMEM = 1024 + TILE * (1 + FWD_STAGES) + 4096 + 256;
  static constexpr int BWDQ_SMEM = 1024 + TILE * 6 + 1024 + 256;  // Q, dO, 2 x {K, V}, lse / D, barriers
  static constexpr int FWD2_STAGES = HD == 128 ? 4 : 6;
  static constexpr int FWD2_SMEM = 1024 + TILE * (2 + FWD2_STAGES) + 4096 + 256;
  // bwd: K, V, two {Q, dO, lse, D} stages, dS^T (128 x 128 bf16)
  static constexpr int BWD_QDO = 2 * TILE + 1024;
  // dQ staging for the TMA reduce-add: the dS^T buffer itself at head_dim 128 (dQ_i is drained after
  // its MMA read dS^T and before the next softmax writes it), its own 32 KB at head_dim 64
  static constexpr int BWD_STAGE = HD == 64 ? 32768 : 0;
  static constexpr int BWD_SMEM_NOPAD = 2 * TILE + 2 * BWD_QDO + 32768 + BWD_STAGE + 256;
  static constexpr int BWD_SMEM = BWD_SMEM_NOPAD + 1024 <= 232448 ? BWD_SMEM_NOPAD + 1024 : BWD_SMEM_NOPAD;
};

// SW128 operand descriptors of a 128-row tile. The MMA issuer builds one base descriptor per tile
// and steps it by constants (the start-address field is the descriptor's low 14 bits, addr >> 4):
// a per-MMA sdesc_sw128 was a ~150-cycle dependent chain on the single issuing thread, longer than
// the 64-cycle 128 x 128 x 16 MMA itself (tools/probes/umma_probe.cu).
//   K-major (rows = M/N, columns = K): k-step kk (16 elements) of the hd dimension
//   MN-major (rows = K):               k-step kk (16 rows)
__device__ __forceinline__ uint64_t kmajor_base(uint32_t addr) { return sdesc_sw128(addr, 16, 1024); }
__device__ __forceinline__ uint64_t mnmajor_base(uint32_t addr) { return sdesc_sw128(addr, 16384, 1024); }
__device__ __forceinline__ uint64_t kmajor_desc(uint64_t base, int kk) {
  return base + static_cast<uint64_t>(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4);
}
__device__ __forceinline__ uint64_t mnmajor_desc(uint64_t base, int kk) { return base + static_cast<uint64_t>(kk * 128); }

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~static_cast<uintptr_t>(1023));
}

// TMEM load / store of N consecutive 32-bit columns of this warp's lane quarter (N = 16 or 32)
template <int N>
__device__ __forceinline__ void tld(uint32_t taddr, uint32_t* r) {
  if constexpr (N == 32) tmem_ld_32x32b_x32(taddr, *reinterpret_cast<uint32_t(*)[32]>(r));
  else tmem_ld_32x32b_x16(taddr, *reinterpret_cast<uint32_t(*)[16]>(r));
}
template <int N>
__device__ __forceinline__ void tst(uint32_t taddr, const uint32_t* r) {
  if constexpr (N == 32) tmem_st_32x32b_x32(taddr, *reinterpret_cast<const uint32_t(*)[32]>(r));
  else if constexpr (N == 16) tmem_st_32x32b_x16(taddr, *reinterpret_cast<const uint32_t(*)[16]>(r));
  else tmem_st_32x32b_x8(taddr, *reinterpret_cast<const uint32_t(*)[8]>(r));
}


template <int HD>
__global__ void __launch_bounds__(kAttnThreads, 1) flash_fwd_kernel(const __grid_constant__ FwdParams p) {
  using Cfg = AttnCfg<HD>;
  constexpr int TILE = Cfg::TILE;
  constexpr int ST = Cfg::FWD_STAGES;
  constexpr uint32_t IDESC_S = idesc_bf16_f32(128, 128, false, false);
  constexpr uint32_t IDESC_O = idesc_bf16_f32(128, HD, false, true);
  constexpr uint32_t O_COL = 256;
  constexpr int OC = HD / 4;  // O columns per softmax warp

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sQ = smem;
  uint8_t* sKV = smem + TILE;
  float* red = reinterpret_cast<float*>(sKV + ST * TILE);  // [2][4 slices][128 rows] partial maxima, then sums
  uint64_t* q_full = reinterpret_cast<uint64_t*>(red + 2 * 4 * 128);
  uint64_t* kv_full = q_full + 1;
  uint64_t* kv_empty = kv_full + ST;
  uint64_t* s_full = kv_empty + ST;
  uint64_t* p_full = s_full + 2;
  uint64_t* o_bar = p_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_bar + 1);

  const int warp = static_cast<int>(warp_uniform(threadIdx.x >> 5));
  const int lane = threadIdx.x & 31;
  const int nbh = p.B * p.nh;
  const int bh = blockIdx.x % nbh;
  const int qb = p.causal ? p.nqb - 1 - static_cast<int>(blockIdx.x) / nbh : static_cast<int>(blockIdx.x) / nbh;
  const int b = bh / p.nh, h = bh % p.nh, g = h / p.rep;
  const int nblk = p.causal ? qb + 1 : p.nqb;
  const int row0 = b * p.S;
  const ProfClock pc{(p.prof & 1) != 0 && blockIdx.x == 0};

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < ST; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[s], kSoftThreads);
    }
    mbar_init(o_bar, 1);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) tma_prefetch(&p.tqkv);
  if (warp == 1) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  pdl_wait();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = warp_uniform(*tmem_slot);

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------------- TMA producer
      mbar_arrive_expect_tx(q_full, TILE);
#pragma unroll
      for (int c = 0; c < HD / 64; ++c) tma_load_2d(sQ + c * 16384, &p.tqkv, q_full, h * HD + c * 64, row0 + qb * 128);
      for (int u = 0; u < 2 * nblk; ++u) {
        const int st = u % ST;
        const long long t0 = pc.now();
        mbar_wait(&kv_empty[st], ((u / ST) & 1) ^ 1);
        pc.add(6, t0);
        mbar_arrive_expect_tx(&kv_full[st], TILE);
        const int col = ((u & 1) ? (p.nh + p.nkv + g) : (p.nh + g)) * HD;
#pragma unroll
        for (int c = 0; c < HD / 64; ++c)
          tma_load_2d(sKV + st * TILE + c * 16384, &p.tqkv, &kv_full[st], col + c * 64, row0 + (u >> 1) * 128);
      }
      pdl_trigger();
    }
  } else if (warp == 1) {
    {
      // ---------------------------------------------------------------- MMA issuer (whole warp, one elected lane issues)
      const ProfClock pm{pc.on && lane == 0};
      mbar_wait(q_full, 0);
      tc_fence_after();
      const uint64_t qa = kmajor_base(smem_u32(sQ));
      const long long tm0 = pm.now();
      auto issue_s = [&](int j) {
        const int u = 2 * j, st = u % ST;
        const long long t0 = pm.now();
        mbar_wait(&kv_full[st], (u / ST) & 1);
        pm.add(1, t0);
        tc_fence_after();
        const uint64_t kb = kmajor_base(smem_u32(sKV + st * TILE));
        const uint32_t d = tmem + static_cast<uint32_t>((j & 1) * 128);
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) umma_bf16_w(d, kmajor_desc(qa, k), kmajor_desc(kb, k), IDESC_S, k > 0 ? 1u : 0u);
        umma_commit_w(&kv_empty[st]);
        umma_commit_w(&s_full[j & 1]);
      };
      issue_s(0);
      for (int j = 0; j < nblk; ++j) {
        if (j + 1 < nblk) issue_s(j + 1);
        long long t0 = pm.now();
        mbar_wait(&p_full[j & 1], (j >> 1) & 1);
        pm.add(0, t0);
        tc_fence_after();
        const int u = 2 * j + 1, st = u % ST;
        t0 = pm.now();
        mbar_wait(&kv_full[st], (u / ST) & 1);
        pm.add(1, t0);
        tc_fence_after();
        const uint64_t vb = mnmajor_base(smem_u32(sKV + st * TILE));
        const uint32_t pa = tmem + static_cast<uint32_t>((j & 1) * 128);
#pragma unroll
        for (int k = 0; k < 8; ++k)
          umma_bf16_ts_w(tmem + O_COL, pa + static_cast<uint32_t>(k * 8), mnmajor_desc(vb, k), IDESC_O,
                       (j > 0 || k > 0) ? 1u : 0u);
        umma_commit_w(&kv_empty[st]);
        umma_commit_w(o_bar);
      }
      pm.add(2, tm0);
    }
  } else {
    // ------------------------------------------------------------------ softmax
    // 16 warps: 4 per TMEM lane quarter (query rows 32 q4 .. 32 q4 + 31), each owning a 32-column
    // slice of the scores (and OC columns of O); row statistics are combined through shared memory
    // with one named barrier per quarter and block.
    const int q4 = warp & 3;
    const int slice = (warp - 2) >> 2;
    const int r = q4 * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    const uint32_t bar_id = 1 + q4;
    const int qpos = qb * 128 + r;
    const float c = p.scale_log2;
    const ProfClock sp{pc.on && threadIdx.x == 64};
    const long long ts0 = sp.now();
    float m_used = 0.f, l = 0.f;  // running max (scaled, log2) and this slice's partial row sum
    for (int j = 0; j < nblk; ++j) {
      const long long t0 = sp.now();
      mbar_wait(&s_full[j & 1], (j >> 1) & 1);
      sp.add(3, t0);
      const long long tc0 = sp.now();
      tc_fence_after();
      const uint32_t sa = tmem + lane_off + static_cast<uint32_t>((j & 1) * 128);
      uint32_t sr[32];
      tld<32>(sa + slice * 32, sr);
      tmem_ld_wait();
      float sv[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) sv[i] = __uint_as_float(sr[i]);
      if (p.causal && j == qb) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (slice * 32 + i > r) sv[i] = -INFINITY;
      }
      // row maximum of the slice: 3-input maxima in 4 independent chains
      float mx[4] = {max3f(sv[0], sv[1], sv[2]), max3f(sv[3], sv[4], sv[5]), max3f(sv[6], sv[7], sv[8]),
                     max3f(sv[9], sv[10], sv[11])};
#pragma unroll
      for (int i = 12; i < 28; i += 8) {
        mx[0] = max3f(mx[0], sv[i], sv[i + 1]);
        mx[1] = max3f(mx[1], sv[i + 2], sv[i + 3]);
        mx[2] = max3f(mx[2], sv[i + 4], sv[i + 5]);
        mx[3] = max3f(mx[3], sv[i + 6], sv[i + 7]);
      }
      float* rb = red + (j & 1) * 512;
      rb[slice * 128 + r] = fmaxf(max3f(mx[0], mx[1], sv[28]), max3f(mx[2], mx[3], fmaxf(sv[29], fmaxf(sv[30], sv[31]))));
      const long long tb0 = sp.now();
      named_bar_sync(bar_id, 128);  // every slice's maximum is in; every S read of the quarter is done
      sp.add(4, tb0);
      const float mrow =
          fmaxf(fmaxf(rb[r], rb[128 + r]), fmaxf(rb[256 + r], rb[384 + r])) * c;
      if (j == 0) {
        m_used = mrow;
      } else if (__any_sync(0xffffffffu, mrow > m_used + kRescaleLog2)) {
        // O and l were accumulated against m_used: rescale once PV_{j-1} has landed in TMEM. The
        // decision is warp-uniform (tcgen05.ld / st are warp-collective: a lane-divergent TMEM access
        // hangs the warp); every lane moves to max(m_used, mrow), a factor of 1 where its max did not
        // grow. The quarter's 4 slice warps see the same rows, so they take the same branch.
        mbar_wait(o_bar, (j - 1) & 1);
        tc_fence_after();
        const float mn = fmaxf(m_used, mrow);
        const float a = ex2_approx(m_used - mn);
        l *= a;
        uint32_t o[OC];
        tld<OC>(tmem + lane_off + O_COL + slice * OC, o);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < OC; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * a);
        tst<OC>(tmem + lane_off + O_COL + slice * OC, o);
        m_used = mn;
      }
      const float nm = -m_used;
      uint32_t pk[16];
      // x = s c - m on packed pairs (FFMA2); 2^x for 6 of the 16 pairs on the FMA pipe (ex2_poly2,
      // FA4-style MUFU offload), the rest on the MUFU; row sums in two packed accumulators (FADD2)
      float2 ls2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float2 x = fma2(make_float2(sv[2 * i], sv[2 * i + 1]), make_float2(c, c), make_float2(nm, nm));
        float2 e;
        if ((i % 8) == 2 || (i % 8) == 5 || (i % 8) == 7) e = ex2_poly2(x);
        else e = make_float2(ex2_approx(x.x), ex2_approx(x.y));
        ls2[i & 1] = add2(ls2[i & 1], e);
        pk[i] = pack_bf16x2(e.x, e.y);
      }
      l += (ls2[0].x + ls2[0].y) + (ls2[1].x + ls2[1].y);
      tst<16>(sa + slice * 16, pk);  // P over S (every S read of this quarter finished at the barrier)
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&p_full[j & 1]);
      sp.add(7, tc0);
    }
    sp.add(5, ts0);
    // ---------------------------------------------------------------- epilogue
    float* rs = red + (nblk & 1) * 512;  // the buffer block nblk - 1 did not use
    rs[slice * 128 + r] = l;
    named_bar_sync(bar_id, 128);
    const float lrow = (rs[r] + rs[128 + r]) + (rs[256 + r] + rs[384 + r]);
    mbar_wait(o_bar, (nblk - 1) & 1);
    tc_fence_after();
    const float inv = 1.f / lrow;
    __nv_bfloat16* orow = p.out + static_cast<long long>(row0 + qpos) * p.ldo + h * HD + slice * OC;
    uint32_t o[OC];
    tld<OC>(tmem + lane_off + O_COL + slice * OC, o);
    tmem_ld_wait();
    uint4* dst = reinterpret_cast<uint4*>(orow);
#pragma unroll
    for (int v = 0; v < OC / 8; ++v) {
      uint4 w;
      w.x = pack_bf16x2(__uint_as_float(o[8 * v + 0]) * inv, __uint_as_float(o[8 * v + 1]) * inv);
      w.y = pack_bf16x2(__uint_as_float(o[8 * v + 2]) * inv, __uint_as_float(o[8 * v + 3]) * inv);
      w.z = pack_bf16x2(__uint_as_float(o[8 * v + 4]) * inv, __uint_as_float(o[8 * v + 5]) * inv);
      w.w = pack_bf16x2(__uint_as_float(o[8 * v + 6]) * inv, __uint_as_float(o[8 * v + 7]) * inv);
      dst[v] = w;
    }
    if (slice == 0) p.lse[(static_cast<long long>(b) * p.nh + h) * p.S + qpos] = m_used + __log2f(lrow);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// Forward, two query tiles per CTA (flash_fwd2_kernel; FA4-style ping-pong): the CTA owns query
// blocks 2p (tile A) and 2p + 1 (tile B) of one (sequence, head) and streams K_j / V_j once for both.
// TMEM holds one S and one O per tile (S_A | S_B | O_A | O_B = 512 columns), so while the softmax
// warps of one tile exponentiate S_t(j), the tensor pipe runs the other tile's P.V and next Q.K^T:
//   S_A(0) S_B(0) | PV_A(0) S_A(1) | PV_B(0) S_B(1) | PV_A(1) S_A(2) | ...
// Softmax: 8 warps per tile, 2 per TMEM lane quarter, each owning a 64-column half of the tile's
// scores (two TMEM loads, one wait) and HD/2 columns of its O; row maxima and sums are combined
// through shared memory with one 64-thread named barrier per quarter and block. Same arithmetic as
// flash_fwd_kernel (packed fp32, lazy warp-uniform O rescale, 3/8 of the exponentials on the FMA
// pipe). S_t(j+1) is issued after PV_t(j) (one S buffer per tile), so a tile's softmax waits one
// P.V + Q.K^T; the other tile's fills the pipe meanwhile. LLaMA shapes (tools/attn_bench.py):
// 8B 94 -> 89 us, 13B 69 -> 64 us, 1B 83 -> 70 us vs the one-tile kernel (PF_ATTN_FWD=1).
template <int HD>
__global__ void __launch_bounds__(kFwd2Threads, 1) flash_fwd2_kernel(const __grid_constant__ FwdParams p) {
  using Cfg = AttnCfg<HD>;
  constexpr int TILE = Cfg::TILE;
  constexpr int ST = Cfg::FWD2_STAGES;
  constexpr uint32_t IDESC_S = idesc_bf16_f32(128, 128, false, false);
  constexpr uint32_t IDESC_O = idesc_bf16_f32(128, HD, false, true);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sQ = smem;  // tile A, tile B
  uint8_t* sKV = smem + 2 * TILE;
  float* red = reinterpret_cast<float*>(sKV + ST * TILE);  // [tile][2 bufs][2 halves][128 rows]
  uint64_t* q_full = reinterpret_cast<uint64_t*>(red + 2 * 2 * 2 * 128);
  uint64_t* kv_full = q_full + 1;
  uint64_t* kv_empty = kv_full + ST;
  uint64_t* s_full = kv_empty + ST;  // [tile]
  uint64_t* p_full = s_full + 2;     // [tile]
  uint64_t* o_bar = p_full + 2;      // [tile]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_bar + 2);

  const int warp = static_cast<int>(warp_uniform(threadIdx.x >> 5));
  const int lane = threadIdx.x & 31;
  const int nbh = p.B * p.nh;
  const int npair = (p.nqb + 1) >> 1;
  const int bh = blockIdx.x % nbh;
  const int pr = p.causal ? npair - 1 - static_cast<int>(blockIdx.x) / nbh : static_cast<int>(blockIdx.x) / nbh;
  const int b = bh / p.nh, h = bh % p.nh, g = h / p.rep;
  const int qbA = 2 * pr, qbB = 2 * pr + 1;
  const bool hasB = qbB < p.nqb;
  const int nA = p.causal ? qbA + 1 : p.nqb;
  const int nB = hasB ? (p.causal ? qbB + 1 : p.nqb) : 0;
  const int nmax = nA > nB ? nA : nB;
  const int row0 = b * p.S;
  const ProfClock pc{(p.prof & 1) != 0 && blockIdx.x == 0};

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < ST; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&s_full[t], 1);
      mbar_init(&p_full[t], 256);
      mbar_init(&o_bar[t], 1);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) tma_prefetch(&p.tqkv);
  if (warp == 1) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  pdl_wait();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = warp_uniform(*tmem_slot);

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------------- TMA producer
      mbar_arrive_expect_tx(q_full, hasB ? 2 * TILE : TILE);
#pragma unroll
      for (int c = 0; c < HD / 64; ++c) {
        tma_load_2d(sQ + c * 16384, &p.tqkv, q_full, h * HD + c * 64, row0 + qbA * 128);
        if (hasB) tma_load_2d(sQ + TILE + c * 16384, &p.tqkv, q_full, h * HD + c * 64, row0 + qbB * 128);
      }
      for (int u = 0; u < 2 * nmax; ++u) {
        const int st = u % ST;
        mbar_wait(&kv_empty[st], ((u / ST) & 1) ^ 1);
        mbar_arrive_expect_tx(&kv_full[st], TILE);
        const int col = ((u & 1) ? (p.nh + p.nkv + g) : (p.nh + g)) * HD;
#pragma unroll
        for (int c = 0; c < HD / 64; ++c)
          tma_load_2d(sKV + st * TILE + c * 16384, &p.tqkv, &kv_full[st], col + c * 64, row0 + (u >> 1) * 128);
      }
      pdl_trigger();
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer (warp-collective issue)
    mbar_wait(q_full, 0);
    tc_fence_after();
    const uint64_t qa0 = kmajor_base(smem_u32(sQ)), qa1 = kmajor_base(smem_u32(sQ + TILE));
    auto issue_s = [&](int t, int j) {  // S_t(j) = Q_t K_j^T; K_j's stage is released by the last tile reading it
      const int u = 2 * j, st = u % ST;
      mbar_wait(&kv_full[st], (u / ST) & 1);
      tc_fence_after();
      const uint64_t kb = kmajor_base(smem_u32(sKV + st * TILE));
#pragma unroll
      for (int k = 0; k < HD / 16; ++k)
        umma_bf16_w(tmem + static_cast<uint32_t>(t * 128), kmajor_desc(t ? qa1 : qa0, k), kmajor_desc(kb, k), IDESC_S,
                    k > 0 ? 1u : 0u);
      umma_commit_w(&s_full[t]);
      if (t == 1 || j >= nB) umma_commit_w(&kv_empty[st]);
    };
    const ProfClock pm{pc.on && lane == 0};
    const long long tm0 = pm.now();
    auto issue_pv = [&](int t, int j) {  // O_t += P_t(j) V_j, P from TMEM over S_t
      const long long t0 = pm.now();
      mbar_wait(&p_full[t], j & 1);
      pm.add(0, t0);
      tc_fence_after();
      const int u = 2 * j + 1, st = u % ST;
      mbar_wait(&kv_full[st], (u / ST) & 1);
      tc_fence_after();
      const uint64_t vb = mnmajor_base(smem_u32(sKV + st * TILE));
#pragma unroll
      for (int k = 0; k < 8; ++k)
        umma_bf16_ts_w(tmem + 256 + static_cast<uint32_t>(t * 128), tmem + static_cast<uint32_t>(t * 128 + k * 8),
                       mnmajor_desc(vb, k), IDESC_O, (j > 0 || k > 0) ? 1u : 0u);
      umma_commit_w(&o_bar[t]);
      if (t == 1 || j >= nB) umma_commit_w(&kv_empty[st]);
    };
    if (nA > 0) issue_s(0, 0);
    if (nB > 0) issue_s(1, 0);
    for (int j = 0; j < nmax; ++j) {
      if (j < nA) {
        issue_pv(0, j);
        if (j + 1 < nA) issue_s(0, j + 1);
      }
      if (j < nB) {
        issue_pv(1, j);
        if (j + 1 < nB) issue_s(1, j + 1);
      }
    }
    pm.add(2, tm0);
  } else {
    // ------------------------------------------------------------------ softmax (8 warps per tile)
    const int q4 = warp & 3;
    const int sw = (warp - 2) >> 2;  // 0..3
    const int t = sw >> 1;           // tile
    const int e = sw & 1;            // 64-column half of the scores, HD/2 columns of O
    const int n_t = t ? nB : nA;
    const int qb = t ? qbB : qbA;
    const int r = q4 * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    const uint32_t bar_id = 1 + t * 4 + q4;
    const uint32_t s_col = tmem + lane_off + static_cast<uint32_t>(t * 128);
    const uint32_t o_col = tmem + lane_off + static_cast<uint32_t>(256 + t * 128 + e * (HD / 2));
    const float c = p.scale_log2;
    float* redt = red + t * 512;
    float m_used = 0.f, l = 0.f;
    const ProfClock sp{pc.on && threadIdx.x == 64};
    const long long ts0 = sp.now();
    for (int j = 0; j < n_t; ++j) {
      long long t0 = sp.now();
      mbar_wait(&s_full[t], j & 1);
      sp.add(3, t0);
      t0 = sp.now();
      tc_fence_after();
      const bool diag = p.causal && j == qb;
      // this warp's 64 scores of the row: two loads, one wait; partial maximum
      uint32_t v[64];
      tld<32>(s_col + e * 64, v);
      tld<32>(s_col + e * 64 + 32, v + 32);
      tmem_ld_wait();
      if (diag) {
#pragma unroll
        for (int i = 0; i < 64; ++i)
          if (e * 64 + i > r) v[i] = __float_as_uint(-INFINITY);
      }
      float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int i = 0; i < 64; i += 8) {
        mx[0] = max3f(mx[0], __uint_as_float(v[i]), __uint_as_float(v[i + 1]));
        mx[1] = max3f(mx[1], __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
        mx[2] = max3f(mx[2], __uint_as_float(v[i + 4]), __uint_as_float(v[i + 5]));
        mx[3] = max3f(mx[3], __uint_as_float(v[i + 6]), __uint_as_float(v[i + 7]));
      }
      float* rb = redt + (j & 1) * 256;
      rb[e * 128 + r] = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
      named_bar_sync(bar_id, 64);  // both halves' maxima are in; both halves' S reads are done
      const float mrow = fmaxf(rb[r], rb[128 + r]) * c;
      sp.add(4, t0);
      t0 = sp.now();
      if (j == 0) {
        m_used = mrow;
      } else if (__any_sync(0xffffffffu, mrow > m_used + kRescaleLog2)) {
        mbar_wait(&o_bar[t], (j - 1) & 1);
        tc_fence_after();
        const float mn = fmaxf(m_used, mrow);
        const float a = ex2_approx(m_used - mn);
        l *= a;
#pragma unroll 1
        for (int c0 = 0; c0 < HD / 2; c0 += 16) {
          uint32_t o[16];
          tld<16>(o_col + c0, o);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * a);
          tst<16>(o_col + c0, o);
        }
        m_used = mn;
      }
      const float nm = -m_used;
      float2 ls2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int q = hf * 32 + 2 * i;
          const float2 x = fma2(make_float2(__uint_as_float(v[q]), __uint_as_float(v[q + 1])), make_float2(c, c),
                                make_float2(nm, nm));
          float2 ev;
          if ((i % 8) == 2 || (i % 8) == 5 || (i % 8) == 7) ev = ex2_poly2(x);
          else ev = make_float2(ex2_approx(x.x), ex2_approx(x.y));
          ls2[i & 1] = add2(ls2[i & 1], ev);
          pk[i] = pack_bf16x2(ev.x, ev.y);
        }
        tst<16>(s_col + e * 32 + hf * 16, pk);  // P (bf16 pairs) over S, after the barrier
      }
      l += (ls2[0].x + ls2[0].y) + (ls2[1].x + ls2[1].y);
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&p_full[t]);
      sp.add(7, t0);
    }
    sp.add(5, ts0);
    if (n_t > 0) {
      // ---------------------------------------------------------------- epilogue of tile t: O / l, LSE
      float* rs = redt + (n_t & 1) * 256;  // the buffer block n_t - 1 did not use
      rs[e * 128 + r] = l;
      named_bar_sync(bar_id, 64);
      const float lrow = rs[r] + rs[128 + r];
      mbar_wait(&o_bar[t], (n_t - 1) & 1);
      tc_fence_after();
      const float inv = 1.f / lrow;
      const int qpos = qb * 128 + r;
      __nv_bfloat16* orow = p.out + static_cast<long long>(row0 + qpos) * p.ldo + h * HD + e * (HD / 2);
#pragma unroll 1
      for (int c0 = 0; c0 < HD / 2; c0 += 16) {
        uint32_t o[16];
        tld<16>(o_col + c0, o);
        tmem_ld_wait();
        uint4* dst = reinterpret_cast<uint4*>(orow + c0);
#pragma unroll
        for (int vv = 0; vv < 2; ++vv) {
          uint4 w;
          w.x = pack_bf16x2(__uint_as_float(o[8 * vv + 0]) * inv, __uint_as_float(o[8 * vv + 1]) * inv);
          w.y = pack_bf16x2(__uint_as_float(o[8 * vv + 2]) * inv, __uint_as_float(o[8 * vv + 3]) * inv);
          w.z = pack_bf16x2(__uint_as_float(o[8 * vv + 4]) * inv, __uint_as_float(o[8 * vv + 5]) * inv);
          w.w = pack_bf16x2(__uint_as_float(o[8 * vv + 6]) * inv, __uint_as_float(o[8 * vv + 7]) * inv);
          dst[vv] = w;
        }
      }
      if (e == 0) p.lse[(static_cast<long long>(b) * p.nh + h) * p.S + qpos] = m_used + __log2f(lrow);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// D[b, h, s] = sum_d dO * O (fp32 from the bf16 tensors); zero the dQ accumulator. HD/8 threads per
// (token, head), 16-byte loads and stores.
template <int HD>
__global__ void flash_bwd_pre_kernel(const __nv_bfloat16* __restrict__ out, const __nv_bfloat16* __restrict__ dout,
                                     float* __restrict__ D, float* __restrict__ dq_acc, int T, int S, int nh) {
  pdl_begin();
  constexpr int TPR = HD / 8;  // threads per row
  const long long n = static_cast<long long>(T) * nh * TPR;
  for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < n;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long w = idx / TPR;  // (token, head)
    const int part = static_cast<int>(idx % TPR);
    const long long off = w * HD + part * 8;
    float o[8], d[8];
    load8(out + off, o);
    load8(dout + off, d);
    float acc = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) acc = fmaf(o[e], d[e], acc);
    if (dq_acc) {  // the fused dQ path accumulates into it (the separate dQ kernel stores it whole)
      float4* z = reinterpret_cast<float4*>(dq_acc + off);
      z[0] = make_float4(0.f, 0.f, 0.f, 0.f);
      z[1] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int o2 = TPR / 2; o2 > 0; o2 >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o2, TPR);
    if (part == 0) {
      const long long t = w / nh;
      const int h = static_cast<int>(w % nh);
      const int b = static_cast<int>(t / S), s = static_cast<int>(t % S);
      D[(static_cast<long long>(b) * nh + h) * S + s] = acc;
    }
  }
}

// P^T and dS^T of 16 queries of a key row (backward softmax): P = 2^(S c - LSE_q), dS = P (dP - D_q), both
// packed to bf16 pairs; LSE / D come from shared memory (lse_s, d_s: 32-bit shared addresses of query q0);
// MASK zeroes queries before the key (the diagonal block of a causal pass)
template <bool MASK>
__device__ __forceinline__ void bwd_half(const uint32_t* sr, const uint32_t* dr, uint32_t lse_s, uint32_t d_s, float c,
                                         int q0, int r, uint32_t (&pk)[8], uint32_t (&dk)[8]) {
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    const float4 L = lds_v4(lse_s + 16 * v), Dd = lds_v4(d_s + 16 * v);
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      // one pair of queries t, t + 1: packed fp32 (FFMA2 / FADD2 / FMUL2); the exponentials of
      // 3 pairs in 8 on the FMA pipe (ex2_poly2), the rest on the MUFU
      const int t = 4 * v + 2 * h2;
      const float2 lq = h2 ? make_float2(-L.z, -L.w) : make_float2(-L.x, -L.y);
      const float2 nd = h2 ? make_float2(-Dd.z, -Dd.w) : make_float2(-Dd.x, -Dd.y);
      const float2 x = fma2(make_float2(__uint_as_float(sr[t]), __uint_as_float(sr[t + 1])), make_float2(c, c), lq);
      float2 pv;
      if ((v * 2 + h2) % 8 == 2 || (v * 2 + h2) % 8 == 5 || (v * 2 + h2) % 8 == 7) pv = ex2_poly2(x);
      else pv = make_float2(ex2_approx(x.x), ex2_approx(x.y));
      if (MASK) {  // key r is after query q0 + t
        if (q0 + t < r) pv.x = 0.f;
        if (q0 + t + 1 < r) pv.y = 0.f;
      }
      const float2 dd = mul2(pv, add2(make_float2(__uint_as_float(dr[t]), __uint_as_float(dr[t + 1])), nd));
      pk[2 * v + h2] = pack_bf16x2(pv.x, pv.y);
      dk[2 * v + h2] = pack_bf16x2(dd.x, dd.y);
    }
  }
}

template <int HD, bool SEP>
__global__ void __launch_bounds__(SEP ? kAttnThreads : kBwdThreads, 1) flash_bwd_kernel(const __grid_constant__ BwdParams p) {
  using Cfg = AttnCfg<HD>;
  constexpr int TILE = Cfg::TILE;
  constexpr uint32_t IDESC_SS = idesc_bf16_f32(128, 128, false, false);  // S^T, dP^T
  constexpr uint32_t IDESC_TS = idesc_bf16_f32(128, HD, false, true);    // dV: A = P^T in TMEM; dK: A = dS^T in smem
                                                                         // (K-major); B MN-major
  constexpr uint32_t IDESC_DQ = idesc_bf16_f32(128, HD, true, true);     // dQ: A (dS) and B (K) MN-major
  // head_dim 128: dQ^T = K^T dS^T instead (M = hd, N = queries; A = K_j and B = dS^T, both MN-major),
  // so a TMEM lane holds one hd column of dQ for all 128 queries and a warp's fp32 reductions into the
  // accumulator are 32 consecutive floats (one 128-byte line) per instruction
  constexpr bool DQ_T = HD == 128;
  constexpr uint32_t IDESC_DQT = idesc_bf16_f32(HD, 128, true, true);
  // TMEM: S^T | dP^T | dV | dK (| dQ when it fits: head_dim 64); at head_dim 128 dQ reuses the dP^T
  // columns (its MMA follows dK's read of dS^T there in issue order)
  constexpr bool DQ_OWN = HD == 64;
  constexpr uint32_t S_COL = 0, DP_COL = 128, DV_COL = 256, DK_COL = 256 + HD;
  constexpr uint32_t DQ_COL = DQ_OWN ? 256 + 2 * HD : DP_COL;
  constexpr int QC = HD / 4;  // dQ columns per softmax warp

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  if constexpr (Cfg::BWD_SMEM == Cfg::BWD_SMEM_NOPAD) {
    if (smem != smem_raw) __trap();  // no room to realign: dynamic shared memory must start 1 KB aligned
  }
  uint8_t* sK = smem;
  uint8_t* sV = smem + TILE;
  uint8_t* sQD = smem + 2 * TILE;  // 2 stages of {Q, dO, lse[128], D[128]}
  uint8_t* sDS = sQD + 2 * Cfg::BWD_QDO;
  uint8_t* sStage = HD == 64 ? sDS + 32768 : sDS;  // dQ staging: 128 rows x 64 fp32
  uint64_t* kv_full = reinterpret_cast<uint64_t*>(sDS + 32768 + Cfg::BWD_STAGE);
  uint64_t* qdo_full = kv_full + 1;
  uint64_t* qdo_empty = qdo_full + 2;
  uint64_t* s_full = qdo_empty + 2;
  uint64_t* p_full = s_full + 1;
  uint64_t* dq_full = p_full + 1;
  uint64_t* dq_empty = dq_full + 1;
  uint64_t* dkv_full = dq_empty + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dkv_full + 1);

  const int warp = static_cast<int>(warp_uniform(threadIdx.x >> 5));
  const int lane = threadIdx.x & 31;
  const int nbg = p.B * p.nkv;
  const int bg = blockIdx.x % nbg;
  const int j = static_cast<int>(blockIdx.x) / nbg;  // causal: key block 0 (the most query blocks) first
  const int b = bg / p.nkv, g = bg % p.nkv;
  const int row0 = b * p.S;
  const int i0 = p.causal ? j : 0;
  const int nq = p.nqb - i0;
  const int niter = p.rep * nq;
  const ProfClock pc{(p.prof & 1) != 0 && blockIdx.x == 0};

  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&qdo_full[s], 1);
      mbar_init(&qdo_empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(p_full, kSoftThreads);
    mbar_init(dq_full, 1);
    mbar_init(dq_empty, 32 * kDrainWarps);
    mbar_init(dkv_full, 1);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&p.tqkv);
    tma_prefetch(&p.tdo);
    tma_prefetch(&p.tdq);
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  pdl_wait();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = warp_uniform(*tmem_slot);

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------------- TMA producer
      mbar_arrive_expect_tx(kv_full, 2 * TILE);
#pragma unroll
      for (int c = 0; c < HD / 64; ++c) {
        tma_load_2d(sK + c * 16384, &p.tqkv, kv_full, (p.nh + g) * HD + c * 64, row0 + j * 128);
        tma_load_2d(sV + c * 16384, &p.tqkv, kv_full, (p.nh + p.nkv + g) * HD + c * 64, row0 + j * 128);
      }
      for (int it = 0; it < niter; ++it) {
        const int st = it & 1;
        const int h = g * p.rep + it % p.rep, i = i0 + it / p.rep;
        mbar_wait(&qdo_empty[st], ((it >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&qdo_full[st], Cfg::BWD_QDO);
        uint8_t* base = sQD + st * Cfg::BWD_QDO;
#pragma unroll
        for (int c = 0; c < HD / 64; ++c) {
          tma_load_2d(base + c * 16384, &p.tqkv, &qdo_full[st], h * HD + c * 64, row0 + i * 128);
          tma_load_2d(base + TILE + c * 16384, &p.tdo, &qdo_full[st], h * HD + c * 64, row0 + i * 128);
        }
        const long long li = (static_cast<long long>(b) * p.nh + h) * p.S + i * 128;
        bulk_load_1d(base + 2 * TILE, p.lse + li, 512, &qdo_full[st]);
        bulk_load_1d(base + 2 * TILE + 512, p.D + li, 512, &qdo_full[st]);
      }
      pdl_trigger();
    }
  } else if (warp == 1) {
    {
      // ---------------------------------------------------------------- MMA issuer (whole warp, one elected lane issues)
      const ProfClock pm{pc.on && lane == 0};
      mbar_wait(kv_full, 0);
      tc_fence_after();
      const uint64_t ka = kmajor_base(smem_u32(sK)), va = kmajor_base(smem_u32(sV));
      const uint64_t ka_mn = mnmajor_base(smem_u32(sK)), dsa = mnmajor_base(smem_u32(sDS));
      const uint64_t dsa_k = kmajor_base(smem_u32(sDS));  // dS^T rows = keys (M), queries = K
      const long long tm0 = pm.now();
      for (int it = 0; it < niter; ++it) {
        const int st = it & 1;
        long long t0 = pm.now();
        mbar_wait(&qdo_full[st], (it >> 1) & 1);
        pm.add(8, t0);
        tc_fence_after();
        const uint32_t qaddr = smem_u32(sQD + st * Cfg::BWD_QDO);
        const uint64_t qa = kmajor_base(qaddr), da = kmajor_base(qaddr + TILE);
        const uint64_t qa_mn = mnmajor_base(qaddr), da_mn = mnmajor_base(qaddr + TILE);
        // S^T = K_j Q_i^T (over P^T of the previous iteration: its dV MMA was issued before)
#pragma unroll
        for (int k = 0; k < HD / 16; ++k)
          umma_bf16_w(tmem + S_COL, kmajor_desc(ka, k), kmajor_desc(qa, k), IDESC_SS, k > 0 ? 1u : 0u);
        if (!SEP && !DQ_OWN && it > 0) {  // dQ_{it-1} (in the dP columns) has been drained
          t0 = pm.now();
          mbar_wait(dq_empty, (it - 1) & 1);
          pm.add(9, t0);
          tc_fence_after();
        }
        // dP^T = V_j dO_i^T
#pragma unroll
        for (int k = 0; k < HD / 16; ++k)
          umma_bf16_w(tmem + DP_COL, kmajor_desc(va, k), kmajor_desc(da, k), IDESC_SS, k > 0 ? 1u : 0u);
        umma_commit_w(s_full);
        t0 = pm.now();
        mbar_wait(p_full, it & 1);
        pm.add(10, t0);
        tc_fence_after();
        // dV += P^T dO_i, dK += dS^T Q_i (A from TMEM, 16 queries per k-step)
#pragma unroll
        for (int k = 0; k < 8; ++k)
          umma_bf16_ts_w(tmem + DV_COL, tmem + S_COL + k * 8, mnmajor_desc(da_mn, k), IDESC_TS, (it > 0 || k > 0) ? 1u : 0u);
#pragma unroll
        for (int k = 0; k < 8; ++k)
          umma_bf16_w(tmem + DK_COL, kmajor_desc(dsa_k, k), mnmajor_desc(qa_mn, k), IDESC_TS, (it > 0 || k > 0) ? 1u : 0u);
        if constexpr (!SEP) {
          if (DQ_OWN && it > 0) {  // dQ_{it-1} has been drained from its own columns
            mbar_wait(dq_empty, (it - 1) & 1);
            tc_fence_after();
          }
          // dQ_i = dS K_j
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if constexpr (DQ_T)
              umma_bf16_w(tmem + DQ_COL, mnmajor_desc(ka_mn, k), mnmajor_desc(dsa, k), IDESC_DQT, k > 0 ? 1u : 0u);
            else
              umma_bf16_w(tmem + DQ_COL, mnmajor_desc(dsa, k), mnmajor_desc(ka_mn, k), IDESC_DQ, k > 0 ? 1u : 0u);
        }
        umma_commit_w(&qdo_empty[st]);
        if constexpr (!SEP) umma_commit_w(dq_full);
      }
      pm.add(11, tm0);
      umma_commit_w(dkv_full);
    }
  } else if (!SEP && warp >= 2 + kSoftWarps) {
    // ------------------------------------------------------------------ dQ drain (4 warps)
    // one warp per TMEM lane quarter: rows = queries of block i; tcgen05.ld of dQ_i, the columns
    // handed back (dq_empty) before the fp32 reductions into the accumulator, which overlap the next
    // iteration's S^T / dP^T MMAs and softmax
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    const ProfClock sp{pc.on && warp == 2 + kSoftWarps + 2 && lane == 0};
    for (int it = 0; it < niter; ++it) {
      const int h = g * p.rep + it % p.rep, i = i0 + it / p.rep;
      long long t0 = sp.now();
      mbar_wait(dq_full, it & 1);
      sp.add(13, t0);
      const long long td0 = sp.now();
      tc_fence_after();
      if constexpr (DQ_T) {
        // lane = hd column d of dQ^T, 32 queries per TMEM load. A 4 x 4 transpose inside each lane quad
        // (two xor-shuffle stages) gives lane 4a + b the 4 consecutive columns 4a .. 4a + 3 of query
        // 4c + b, so a warp's reduction is one red.global.add.v4.f32 per 4 queries (4 x 128 B lines)
        // instead of one scalar red per query: a quarter of the L2 reduction operations
        const int a4 = lane >> 2, b4 = lane & 3;
        float* dst = p.dq_acc + static_cast<long long>(row0 + i * 128) * (p.nh * HD) + h * HD + q4 * 32 + 4 * a4;
        const long long ld = static_cast<long long>(p.nh) * HD;
#pragma unroll
        for (int c0 = 0; c0 < 128; c0 += 32) {
          uint32_t v[32];
          tld<32>(tmem + lane_off + DQ_COL + c0, v);
          tmem_ld_wait();
          if (c0 == 96) {
            tc_fence_before();
            mbar_arrive(dq_empty);
            sp.add(22, td0);
          }
          if (p.prof & 2) continue;  // development: PF_ATTN_PROF=3 drops the dQ reductions (timing only)
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            float x0 = __uint_as_float(v[4 * c]), x1 = __uint_as_float(v[4 * c + 1]);
            float x2 = __uint_as_float(v[4 * c + 2]), x3 = __uint_as_float(v[4 * c + 3]);
            {  // 2 x 2 blocks across lanes b, b ^ 2
              const bool up = (b4 & 2) != 0;
              const float r0 = __shfl_xor_sync(0xffffffffu, up ? x0 : x2, 2);
              const float r1 = __shfl_xor_sync(0xffffffffu, up ? x1 : x3, 2);
              if (up) {
                x0 = r0;
                x1 = r1;
              } else {
                x2 = r0;
                x3 = r1;
              }
            }
            {  // within the 2 x 2 blocks, lanes b, b ^ 1
              const bool up = (b4 & 1) != 0;
              const float r0 = __shfl_xor_sync(0xffffffffu, up ? x0 : x1, 1);
              const float r1 = __shfl_xor_sync(0xffffffffu, up ? x2 : x3, 1);
              if (up) {
                x0 = r0;
                x2 = r1;
              } else {
                x1 = r0;
                x3 = r1;
              }
            }
            red_add_v4(dst + (c0 + 4 * c + b4) * ld, x0, x1, x2, x3);
          }
        }
        sp.add(15, td0);
        continue;
      }
      // 64 columns at a time: TMEM -> this warp's 32 staged rows as two 32 x 32 fp32 SWIZZLE_128B boxes
      // (16-byte chunk c of row l at c ^ (l % 8): 4-way instead of 32-way bank conflicts) -> TMA
      // reduce-add of each box into the accumulator
      uint8_t* stage = sStage + q4 * 8192;
#pragma unroll
      for (int c0 = 0; c0 < HD; c0 += 64) {
        uint32_t v[64];
        tld<32>(tmem + lane_off + DQ_COL + c0, v);
        tld<32>(tmem + lane_off + DQ_COL + c0 + 32, v + 32);
        tmem_ld_wait();
        if (c0 > 0) {  // the previous boxes' reduces have finished reading the staging rows
          if (lane == 0) bulk_wait_read0();
          __syncwarp();
        }
#pragma unroll
        for (int bx = 0; bx < 2; ++bx) {
          uint8_t* srow = stage + bx * 4096 + lane * 128;
#pragma unroll
          for (int ch = 0; ch < 8; ++ch)
            *reinterpret_cast<uint4*>(srow + ((ch ^ (lane & 7)) << 4)) =
                make_uint4(v[bx * 32 + 4 * ch], v[bx * 32 + 4 * ch + 1], v[bx * 32 + 4 * ch + 2], v[bx * 32 + 4 * ch + 3]);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_reduce_add_2d(&p.tdq, stage, h * HD + c0, row0 + i * 128 + q4 * 32);
          tma_reduce_add_2d(&p.tdq, stage + 4096, h * HD + c0 + 32, row0 + i * 128 + q4 * 32);
          bulk_commit();
        }
      }
      if (lane == 0) bulk_wait_read0();  // staging free for the next softmax (head_dim 128: it is dS^T)
      __syncwarp();
      tc_fence_before();
      mbar_arrive(dq_empty);
      sp.add(22, td0);
      sp.add(15, td0);
    }
    if (lane == 0) bulk_wait0();  // every reduce-add has landed before the CTA retires
  } else {
    // ------------------------------------------------------------------ softmax, then dK dV
    // 16 warps: 4 per TMEM lane quarter, each owning 32 query columns of S^T / dP^T and a share of
    // the final dK / dV rows.
    const int q4 = warp & 3;
    const int slice = (warp - 2) >> 2;
    const int r = q4 * 32 + lane;  // key row of S^T
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    const uint32_t bar_id = 1 + q4;
    const float c = p.scale_log2;
    const uint32_t ds_row = smem_u32(sDS + (slice >> 1) * 16384 + r * 128);
    const ProfClock sp{pc.on && threadIdx.x == 64};
    const long long ts0 = sp.now();
    for (int it = 0; it < niter; ++it) {
      const int i = i0 + it / p.rep;
      const int st = it & 1;
      mbar_wait(&qdo_full[st], (it >> 1) & 1);  // lse / D of this query block are in shared memory
      // lse[128] then D[128] of this query block, this slice's 32 queries
      const uint32_t lse_s = smem_u32(sQD + st * Cfg::BWD_QDO + 2 * TILE) + slice * 128;
      long long t0 = sp.now();
      mbar_wait(s_full, it & 1);
      sp.add(12, t0);
      const long long tc0 = sp.now();
      tc_fence_after();
      uint32_t sr[32];
      tld<32>(tmem + lane_off + S_COL + slice * 32, sr);
      tmem_ld_wait();
      sp.add(18, tc0);
      t0 = sp.now();
      named_bar_sync(bar_id, 128);  // every S^T read of the quarter is done before P^T goes over it
      sp.add(17, t0);
      const bool diag = p.causal && i == j;
      const long long tt0 = sp.now();
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        uint32_t dr[16], pk[8], dk[8];
        tld<16>(tmem + lane_off + DP_COL + slice * 32 + hf * 16, dr);
        tmem_ld_wait();
        if (diag) bwd_half<true>(sr + hf * 16, dr, lse_s + hf * 64, lse_s + 512 + hf * 64, c, slice * 32 + hf * 16, r, pk, dk);
        else bwd_half<false>(sr + hf * 16, dr, lse_s + hf * 64, lse_s + 512 + hf * 64, c, slice * 32 + hf * 16, r, pk, dk);
        tst<8>(tmem + lane_off + S_COL + slice * 16 + hf * 8, pk);
        // dS^T row r, queries [32 slice + 16 hf, +16): region slice/2, 16-byte units (slice%2)*4 + 2 hf .. +2, SW128
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int unit = ((slice & 1) * 4 + hf * 2 + u) ^ (r & 7);
          sts_v4(ds_row + unit * 16, make_uint4(dk[4 * u], dk[4 * u + 1], dk[4 * u + 2], dk[4 * u + 3]));
        }
      }
      sp.add(19, tt0);
      sp.add(20, tt0);
      const long long tw0 = sp.now();
      tmem_st_wait();
      sp.add(21, tw0);
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(p_full);
      sp.add(14, tc0);
    }
    sp.add(16, ts0);
    // ---------------------------------------------------------------- dK, dV of key block j
    mbar_wait(dkv_full, 0);
    tc_fence_after();
    const int pos = j * 128 + r;
    __nv_bfloat16* row = p.dqkv + static_cast<long long>(row0 + pos) * p.ldq;
    if (slice >= 2) {  // dV: slices 2, 3 take HD/2 columns each
      constexpr int VC = HD / 2;
#pragma unroll
      for (int c0 = 0; c0 < VC; c0 += 32) {
        const int col = (slice - 2) * VC + c0;
        uint32_t w[32];
        tld<32>(tmem + lane_off + DV_COL + col, w);
        tmem_ld_wait();
        uint4* dv = reinterpret_cast<uint4*>(row + (p.nh + p.nkv + g) * HD + col);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          dv[u] = make_uint4(pack_bf16x2(__uint_as_float(w[8 * u]), __uint_as_float(w[8 * u + 1])),
                             pack_bf16x2(__uint_as_float(w[8 * u + 2]), __uint_as_float(w[8 * u + 3])),
                             pack_bf16x2(__uint_as_float(w[8 * u + 4]), __uint_as_float(w[8 * u + 5])),
                             pack_bf16x2(__uint_as_float(w[8 * u + 6]), __uint_as_float(w[8 * u + 7])));
      }
    } else {  // dK: slices 0, 1 take HD/4 columns of the first half each and their RoPE partners
      constexpr int KC = HD / 4;
#pragma unroll
      for (int c16 = 0; c16 < KC; c16 += 16) {
        const int col = slice * KC + c16;
        uint32_t a[16], bb[16];
        tld<16>(tmem + lane_off + DK_COL + col, a);
        tld<16>(tmem + lane_off + DK_COL + HD / 2 + col, bb);
        tmem_ld_wait();
        const float2* cs = p.rope ? p.rope + static_cast<long long>(pos) * (HD / 2) + col : nullptr;
        float fa[16], fb[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float ga = __uint_as_float(a[e]) * p.scale, gb = __uint_as_float(bb[e]) * p.scale;
          if (cs) {
            const float2 t = cs[e];
            fa[e] = ga * t.x + gb * t.y;
            fb[e] = gb * t.x - ga * t.y;
          } else {
            fa[e] = ga;
            fb[e] = gb;
          }
        }
        uint4* ka = reinterpret_cast<uint4*>(row + (p.nh + g) * HD + col);
        uint4* kb = reinterpret_cast<uint4*>(row + (p.nh + g) * HD + HD / 2 + col);
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          ka[u] = make_uint4(pack_bf16x2(fa[8 * u], fa[8 * u + 1]), pack_bf16x2(fa[8 * u + 2], fa[8 * u + 3]),
                             pack_bf16x2(fa[8 * u + 4], fa[8 * u + 5]), pack_bf16x2(fa[8 * u + 6], fa[8 * u + 7]));
          kb[u] = make_uint4(pack_bf16x2(fb[8 * u], fb[8 * u + 1]), pack_bf16x2(fb[8 * u + 2], fb[8 * u + 3]),
                             pack_bf16x2(fb[8 * u + 4], fb[8 * u + 5]), pack_bf16x2(fb[8 * u + 6], fb[8 * u + 7]));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// dq = scale * dQ_acc with the RoPE backward, bf16 into dqkv's q columns. One thread per
// (token, head, pair d < HD/2).
// dQ without atomics (flash_bwd_q_kernel, PF_ATTN_BWD=2; run before the dK / dV kernel, which then
// has no dQ work): one CTA per (sequence, head, 128-query block) loops over the key blocks the queries see,
// recomputing S = Q K_j^T and dP = dO V_j^T (TMEM: S in two buffers | dP | dQ), P = 2^(S c - LSE),
// dS = P (dP - D) as bf16 over S, and dQ += dS K_j with A = dS from TMEM. dQ stays in TMEM for the
// whole loop and leaves once, unscaled fp32, into dq_acc (plain stores: the CTA owns its rows);
// flash_bwd_dq_kernel scales it, applies the RoPE backward and writes dq into dqkv after the dK / dV
// kernel has consumed q. S(j + 2) reuses S(j)'s buffer after dQ(j) read dS(j); dP(j + 1) follows
// the softmax's read of dP(j). The softmax warps (4 per TMEM lane quarter, lane = query row, 32
// key columns each) write dS over the first 16 of their own 32 S columns: no cross-warp hazard.
template <int HD>
__global__ void __launch_bounds__(kAttnThreads, 1) flash_bwd_q_kernel(const __grid_constant__ BwdParams p) {
  using Cfg = AttnCfg<HD>;
  constexpr int TILE = Cfg::TILE;
  constexpr uint32_t IDESC_SS = idesc_bf16_f32(128, 128, false, false);  // S, dP: A (Q, dO) and B (K, V) K-major
  constexpr uint32_t IDESC_DQ = idesc_bf16_f32(128, HD, false, true);    // dQ: A = dS in TMEM, B = K_j MN-major
  constexpr uint32_t DP_COL = 256, DQ_COL = 384;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sQ = smem;
  uint8_t* sDO = smem + TILE;
  uint8_t* sKV = smem + 2 * TILE;  // 2 stages of {K_j, V_j}
  float* sLD = reinterpret_cast<float*>(sKV + 4 * TILE);  // lse[128], D[128]
  uint64_t* qd_full = reinterpret_cast<uint64_t*>(sLD + 256);
  uint64_t* kv_full = qd_full + 1;   // [2]
  uint64_t* kv_empty = kv_full + 2;  // [2]
  uint64_t* s_full = kv_empty + 2;   // [2] per S buffer
  uint64_t* dp_full = s_full + 2;
  uint64_t* p_full = dp_full + 1;
  uint64_t* dq_done = p_full + 1;
  uint64_t* dp_read = dq_done + 1;  // the softmax has dP(j) in registers: dP(j + 1) may go over it
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dp_read + 1);

  const int warp = static_cast<int>(warp_uniform(threadIdx.x >> 5));
  const int lane = threadIdx.x & 31;
  const int nbh = p.B * p.nh;
  const int bh = blockIdx.x % nbh;
  const int i = p.causal ? p.nqb - 1 - static_cast<int>(blockIdx.x) / nbh : static_cast<int>(blockIdx.x) / nbh;
  const int b = bh / p.nh, h = bh % p.nh, g = h / p.rep;
  const int nblk = p.causal ? i + 1 : p.nqb;
  const int row0 = b * p.S;

  if (threadIdx.x == 0) {
    mbar_init(qd_full, 1);
    for (int s2 = 0; s2 < 2; ++s2) {
      mbar_init(&kv_full[s2], 1);
      mbar_init(&kv_empty[s2], 1);
      mbar_init(&s_full[s2], 1);
    }
    mbar_init(dp_full, 1);
    mbar_init(p_full, kSoftThreads);
    mbar_init(dq_done, 1);
    mbar_init(dp_read, kSoftThreads);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&p.tqkv);
    tma_prefetch(&p.tdo);
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  pdl_wait();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = warp_uniform(*tmem_slot);

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------------- TMA producer
      mbar_arrive_expect_tx(qd_full, 2 * TILE + 1024);
#pragma unroll
      for (int c = 0; c < HD / 64; ++c) {
        tma_load_2d(sQ + c * 16384, &p.tqkv, qd_full, h * HD + c * 64, row0 + i * 128);
        tma_load_2d(sDO + c * 16384, &p.tdo, qd_full, h * HD + c * 64, row0 + i * 128);
      }
      const long long li = (static_cast<long long>(b) * p.nh + h) * p.S + i * 128;
      bulk_load_1d(sLD, p.lse + li, 512, qd_full);
      bulk_load_1d(sLD + 128, p.D + li, 512, qd_full);
      for (int j = 0; j < nblk; ++j) {
        const int st = j & 1;
        mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&kv_full[st], 2 * TILE);
        uint8_t* base = sKV + st * 2 * TILE;
#pragma unroll
        for (int c = 0; c < HD / 64; ++c) {
          tma_load_2d(base + c * 16384, &p.tqkv, &kv_full[st], (p.nh + g) * HD + c * 64, row0 + j * 128);
          tma_load_2d(base + TILE + c * 16384, &p.tqkv, &kv_full[st], (p.nh + p.nkv + g) * HD + c * 64,
                      row0 + j * 128);
        }
      }
      pdl_trigger();
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer (warp-collective issue)
    mbar_wait(qd_full, 0);
    tc_fence_after();
    const uint64_t qa = kmajor_base(smem_u32(sQ)), da = kmajor_base(smem_u32(sDO));
    auto issue_s = [&](int j) {
      const int st = j & 1;
      mbar_wait(&kv_full[st], (j >> 1) & 1);
      tc_fence_after();
      const uint64_t kb = kmajor_base(smem_u32(sKV + st * 2 * TILE));
#pragma unroll
      for (int k = 0; k < HD / 16; ++k)
        umma_bf16_w(tmem + static_cast<uint32_t>(st * 128), kmajor_desc(qa, k), kmajor_desc(kb, k), IDESC_SS,
                    k > 0 ? 1u : 0u);
      umma_commit_w(&s_full[st]);
    };
    auto issue_dp = [&](int j) {
      const int st = j & 1;
      mbar_wait(&kv_full[st], (j >> 1) & 1);
      tc_fence_after();
      const uint64_t vb = kmajor_base(smem_u32(sKV + st * 2 * TILE + TILE));
#pragma unroll
      for (int k = 0; k < HD / 16; ++k)
        umma_bf16_w(tmem + DP_COL, kmajor_desc(da, k), kmajor_desc(vb, k), IDESC_SS, k > 0 ? 1u : 0u);
      umma_commit_w(dp_full);
    };
    issue_s(0);
    issue_dp(0);
    if (nblk > 1) issue_s(1);
    for (int j = 0; j < nblk; ++j) {
      const int st = j & 1;
      if (j + 1 < nblk) {  // dP(j + 1) under softmax(j), as soon as the softmax holds dP(j)
        mbar_wait(dp_read, j & 1);
        tc_fence_after();
        issue_dp(j + 1);
      }
      mbar_wait(p_full, j & 1);  // dS(j) is in TMEM over S(j)
      tc_fence_after();
      // dQ += dS(j) K_j: 16 keys per k-step, key slice kk / 2's first 16 columns of S(j)
      const uint64_t kb_mn = mnmajor_base(smem_u32(sKV + st * 2 * TILE));
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        umma_bf16_ts_w(tmem + DQ_COL, tmem + static_cast<uint32_t>(st * 128 + (kk >> 1) * 32 + (kk & 1) * 8),
                       mnmajor_desc(kb_mn, kk), IDESC_DQ, (j > 0 || kk > 0) ? 1u : 0u);
      umma_commit_w(&kv_empty[st]);  // K_j, V_j: dP(j) and dQ(j) were their last readers
      if (j + 2 < nblk) issue_s(j + 2);
    }
    umma_commit_w(dq_done);
  } else {
    // ------------------------------------------------------------------ softmax (16 warps)
    const int q4 = warp & 3;
    const int slice = (warp - 2) >> 2;
    const int r = q4 * 32 + lane;  // query row
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    const float c = p.scale_log2;
    mbar_wait(qd_full, 0);
    const float2 nl = make_float2(-sLD[r], -sLD[r]);
    const float2 nd = make_float2(-sLD[128 + r], -sLD[128 + r]);
    for (int j = 0; j < nblk; ++j) {
      const int st = j & 1;
      mbar_wait(&s_full[st], (j >> 1) & 1);
      mbar_wait(dp_full, j & 1);
      tc_fence_after();
      uint32_t sr[32], dr[32];
      tld<32>(tmem + lane_off + static_cast<uint32_t>(st * 128 + slice * 32), sr);
      tld<32>(tmem + lane_off + DP_COL + static_cast<uint32_t>(slice * 32), dr);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(dp_read);
      const bool diag = p.causal && j == i;
      uint32_t pk[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const float2 x = fma2(make_float2(__uint_as_float(sr[2 * e]), __uint_as_float(sr[2 * e + 1])),
                              make_float2(c, c), nl);
        float2 pv;
        if ((e % 8) == 2 || (e % 8) == 5 || (e % 8) == 7) pv = ex2_poly2(x);
        else pv = make_float2(ex2_approx(x.x), ex2_approx(x.y));
        if (diag) {  // key after query
          if (slice * 32 + 2 * e > r) pv.x = 0.f;
          if (slice * 32 + 2 * e + 1 > r) pv.y = 0.f;
        }
        const float2 ds = mul2(pv, add2(make_float2(__uint_as_float(dr[2 * e]), __uint_as_float(dr[2 * e + 1])), nd));
        pk[e] = pack_bf16x2(ds.x, ds.y);
      }
      tst<16>(tmem + lane_off + static_cast<uint32_t>(st * 128 + slice * 32), pk);  // dS over this slice's S
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(p_full);
    }
    // ---------------------------------------------------------------- dQ (unscaled fp32) -> dq_acc
    mbar_wait(dq_done, 0);
    tc_fence_after();
    constexpr int QC = HD / 4;
    float* dst = p.dq_acc + static_cast<long long>(row0 + i * 128 + r) * (p.nh * HD) + h * HD + slice * QC;
#pragma unroll
    for (int c0 = 0; c0 < QC; c0 += 16) {
      uint32_t v[16];
      tld<16>(tmem + lane_off + DQ_COL + static_cast<uint32_t>(slice * QC + c0), v);
      tmem_ld_wait();
      float4* d4 = reinterpret_cast<float4*>(dst + c0);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        d4[u] = make_float4(__uint_as_float(v[4 * u]), __uint_as_float(v[4 * u + 1]), __uint_as_float(v[4 * u + 2]),
                            __uint_as_float(v[4 * u + 3]));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

template <int HD>
__global__ void flash_bwd_dq_kernel(const float* __restrict__ dq_acc, __nv_bfloat16* __restrict__ dqkv, long long ldq,
                                    const float2* __restrict__ rope, int T, int S, int nh, float scale) {
  pdl_begin();
  constexpr int HALF = HD / 2;
  const long long n = static_cast<long long>(T) * nh * (HALF / 4);
  for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < n;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int d4 = static_cast<int>(idx % (HALF / 4)) * 4;
    const long long th = idx / (HALF / 4);
    const long long t = th / nh;
    const int h = static_cast<int>(th % nh);
    const float* src = dq_acc + t * nh * HD + h * HD;
    const float4 a = *reinterpret_cast<const float4*>(src + d4);
    const float4 c = *reinterpret_cast<const float4*>(src + HALF + d4);
    float ga[4] = {a.x * scale, a.y * scale, a.z * scale, a.w * scale};
    float gb[4] = {c.x * scale, c.y * scale, c.z * scale, c.w * scale};
    float oa[4], ob[4];
    const float2* cs = rope ? rope + static_cast<long long>(t % S) * HALF + d4 : nullptr;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (cs) {
        const float2 r = cs[e];
        oa[e] = ga[e] * r.x + gb[e] * r.y;
        ob[e] = gb[e] * r.x - ga[e] * r.y;
      } else {
        oa[e] = ga[e];
        ob[e] = gb[e];
      }
    }
    __nv_bfloat16* dst = dqkv + t * ldq + h * HD;
    *reinterpret_cast<uint2*>(dst + d4) = make_uint2(pack_bf16x2(oa[0], oa[1]), pack_bf16x2(oa[2], oa[3]));
    *reinterpret_cast<uint2*>(dst + HALF + d4) = make_uint2(pack_bf16x2(ob[0], ob[1]), pack_bf16x2(ob[2], ob[3]));
  }
}

// PF_ATTN_BWD=2: the separate dQ kernel (flash_bwd_q_kernel, no fp32 atomics) + the dK / dV kernel
// without dQ, instead of the default dK / dV / dQ kernel with fp32 reductions. Measured slower at the
// LLaMA shapes (8B: 143 + 169 us + 35 us of pre / convert vs 335-340 us; both kernels ~40% tensor
// active: S / dP -> softmax -> MMA stays serial in each), kept for A/B
// (profiles/r2_attention_experiments.md).
bool bwd_fused_dq() {
  static const bool fused = [] {
    const char* e = std::getenv("PF_ATTN_BWD");
    return !(e && e[0] == '2');
  }();
  return fused;
}

// PF_ATTN_FWD=1: the one-tile forward (flash_fwd_kernel) instead of the two-tile ping-pong (A/B)
bool fwd_one_tile() {
  static const bool one = [] {
    const char* e = std::getenv("PF_ATTN_FWD");
    return e && e[0] == '1';
  }();
  return one;
}

int attn_prof_enabled() {
  static const int on = [] {
    const char* e = std::getenv("PF_ATTN_PROF");
    return e ? std::atoi(e) : 0;
  }();
  return on;
}

template <int HD>
int fwd_impl(const __nv_bfloat16* qkv, __nv_bfloat16* out, long long ldo, float* lse, int B, int S, int nh, int nkv,
             float scale, bool causal, cudaStream_t s) {
  using Cfg = AttnCfg<HD>;
  FwdParams p{};
  const long long W = static_cast<long long>(nh + 2 * nkv) * HD;
  const long long T = static_cast<long long>(B) * S;
  if (tma_desc_bf16_2d(&p.tqkv, qkv, T, W, W, 64, 128)) return PF_ERR_INVALID;
  p.out = out;
  p.ldo = ldo;
  p.lse = lse;
  p.B = B;
  p.S = S;
  p.nh = nh;
  p.nkv = nkv;
  p.rep = nh / nkv;
  p.nqb = S / 128;
  p.causal = causal ? 1 : 0;
  p.prof = attn_prof_enabled();
  p.scale_log2 = scale * 1.4426950408889634f;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(flash_fwd_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::FWD_SMEM) !=
            cudaSuccess ||
        cudaFuncSetAttribute(flash_fwd2_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::FWD2_SMEM) !=
            cudaSuccess)
      return PF_ERR_CUDA;
    attr = true;
  }
  if (fwd_one_tile())
    launch_k(flash_fwd_kernel<HD>, dim3(B * nh * p.nqb), dim3(kAttnThreads), Cfg::FWD_SMEM, s, p);
  else
    launch_k(flash_fwd2_kernel<HD>, dim3(B * nh * ((p.nqb + 1) / 2)), dim3(kFwd2Threads), Cfg::FWD2_SMEM, s, p);
  return status();
}

template <int HD>
int bwd_impl(const __nv_bfloat16* qkv, const __nv_bfloat16* out, const __nv_bfloat16* dout, const float* lse,
             float* D, float* dq_acc, __nv_bfloat16* dqkv, const float2* rope, int B, int S, int nh, int nkv,
             float scale, bool causal, cudaStream_t s) {
  using Cfg = AttnCfg<HD>;
  const int T = B * S;
  const bool sep = !bwd_fused_dq();
  launch_k(flash_bwd_pre_kernel<HD>, dim3(grid_for(static_cast<long long>(T) * nh * (HD / 8) / 256 + 1)), dim3(256), 0, s,
           out, dout, D, sep ? nullptr : dq_acc, T, S, nh);
  int rc = status();
  if (rc) return rc;
  BwdParams p{};
  const long long W = static_cast<long long>(nh + 2 * nkv) * HD;
  if (tma_desc_bf16_2d(&p.tqkv, qkv, T, W, W, 64, 128)) return PF_ERR_INVALID;
  if (tma_desc_bf16_2d(&p.tdo, dout, T, static_cast<long long>(nh) * HD, static_cast<long long>(nh) * HD, 64, 128))
    return PF_ERR_INVALID;
  if (tma_desc_f32_2d(&p.tdq, dq_acc, T, static_cast<long long>(nh) * HD, static_cast<long long>(nh) * HD, 32, 32))
    return PF_ERR_INVALID;
  p.lse = lse;
  p.D = D;
  p.dq_acc = dq_acc;
  p.dqkv = dqkv;
  p.ldq = W;
  p.rope = rope;
  p.B = B;
  p.S = S;
  p.nh = nh;
  p.nkv = nkv;
  p.rep = nh / nkv;
  p.nqb = S / 128;
  p.causal = causal ? 1 : 0;
  p.prof = attn_prof_enabled();
  p.scale_log2 = scale * 1.4426950408889634f;
  p.scale = scale;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(flash_bwd_kernel<HD, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             Cfg::BWD_SMEM) != cudaSuccess ||
        cudaFuncSetAttribute(flash_bwd_kernel<HD, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             Cfg::BWD_SMEM) != cudaSuccess ||
        cudaFuncSetAttribute(flash_bwd_q_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::BWDQ_SMEM) !=
            cudaSuccess)
      return PF_ERR_CUDA;
    attr = true;
  }
  if (sep) {
    // dQ first (it reads k / v, which the dK / dV kernel overwrites in place), then dK / dV
    launch_k(flash_bwd_q_kernel<HD>, dim3(B * nh * p.nqb), dim3(kAttnThreads), Cfg::BWDQ_SMEM, s, p);
    if ((rc = status())) return rc;
    launch_k(flash_bwd_kernel<HD, true>, dim3(B * nkv * p.nqb), dim3(kAttnThreads), Cfg::BWD_SMEM, s, p);
  } else {
    launch_k(flash_bwd_kernel<HD, false>, dim3(B * nkv * p.nqb), dim3(kBwdThreads), Cfg::BWD_SMEM, s, p);
  }
  if ((rc = status())) return rc;
  launch_k(flash_bwd_dq_kernel<HD>, dim3(grid_for(static_cast<long long>(T) * nh * HD / 8 / 256 + 1)), dim3(256), 0, s,
           dq_acc, dqkv, W, rope, T, S, nh, scale);
  return status();
}

bool shape_ok(int B, int S, int nh, int nkv, int hd) {
  return B > 0 && S > 0 && S % 128 == 0 && nkv > 0 && nh % nkv == 0 && (hd == 64 || hd == 128);
}

}  // namespace

// cycle accounting of the first CTA (PF_ATTN_PROF=1): copy out and reset
int flash_attn_prof_read(unsigned long long* out32) {
  if (cudaMemcpyFromSymbol(out32, g_attn_prof, 32 * sizeof(unsigned long long)) != cudaSuccess) return PF_ERR_CUDA;
  static const unsigned long long zeros[32] = {};
  return cudaMemcpyToSymbol(g_attn_prof, zeros, sizeof(zeros)) == cudaSuccess ? PF_OK : PF_ERR_CUDA;
}

int launch_flash_attn_fwd(const __nv_bfloat16* qkv, __nv_bfloat16* out, long long ldo, float* lse, int B, int S,
                          int nh, int nkv, int hd, float scale, bool causal, cudaStream_t s) {
  if (!shape_ok(B, S, nh, nkv, hd) || ldo % 8) return PF_ERR_INVALID;
  return hd == 128 ? fwd_impl<128>(qkv, out, ldo, lse, B, S, nh, nkv, scale, causal, s)
                   : fwd_impl<64>(qkv, out, ldo, lse, B, S, nh, nkv, scale, causal, s);
}

int launch_flash_attn_bwd(const __nv_bfloat16* qkv, const __nv_bfloat16* out, const __nv_bfloat16* dout,
                          const float* lse, float* D, float* dq_acc, __nv_bfloat16* dqkv, const float2* rope, int B,
                          int S, int nh, int nkv, int hd, float scale, bool causal, cudaStream_t s) {
  if (!shape_ok(B, S, nh, nkv, hd)) return PF_ERR_INVALID;
  return hd == 128 ? bwd_impl<128>(qkv, out, dout, lse, D, dq_acc, dqkv, rope, B, S, nh, nkv, scale, causal, s)
                   : bwd_impl<64>(qkv, out, dout, lse, D, dq_acc, dqkv, rope, B, S, nh, nkv, scale, causal, s);
}

}  // namespace pf
