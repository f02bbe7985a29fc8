// extern "C" wrappers for the standalone kernels (include/pf_device.h).
#include <cuda_runtime.h>

#include <string>

#include "pf_device.h"
#include "pf_device_internal.hpp"

namespace {
thread_local std::string g_last_error;
int record(int rc) {
  if (rc == PF_ERR_CUDA) {
    cudaError_t e = cudaGetLastError();
    g_last_error = cudaGetErrorString(e);
  }
  return rc;
}
}  // namespace

extern "C" {

int pf_gemm_bf16(const void* A, int a_mn_major, long long lda, const void* B, int b_mn_major,
                 long long ldb, void* C, long long ldc, int M, int N, int K, float alpha,
                 int epilogue, int block_n, int* unit_stamp, int stamp, void* stream) {
  if (!A || !B || !C) return PF_ERR_INVALID;
  pf::GemmOperand a{A, lda, a_mn_major != 0};
  pf::GemmOperand b{B, ldb, b_mn_major != 0};
  pf::GemmOut c{C, ldc, unit_stamp, 0, stamp};
  if (block_n == 512)  // CTA-pair kernel, 256 x 256 tiles
    return record(pf::gemm_bf16_pair(a, b, c, M, N, K, alpha, epilogue, static_cast<cudaStream_t>(stream)));
  return record(pf::gemm_bf16(a, b, c, M, N, K, alpha, epilogue, block_n,
                              static_cast<cudaStream_t>(stream)));
}

int pf_gemm_dw_units(const void* A, int a_mn_major, long long lda, const void* B, int b_mn_major,
                     long long ldb, float* G, long long ldg, int M, int N, int K, float alpha,
                     const int* unit_list, const int* unit_count, int max_units,
                     int* unit_stamp, int stamp_offset, int stamp, void* stream) {
  if (!A || !B || !G) return PF_ERR_INVALID;
  pf::GemmOperand a{A, lda, a_mn_major != 0};
  pf::GemmOperand b{B, ldb, b_mn_major != 0};
  pf::GemmOut c{G, ldg, unit_stamp, stamp_offset, stamp};
  return record(pf::gemm_bf16_units(a, b, c, M, N, K, alpha, unit_list, unit_count, max_units,
                                    static_cast<cudaStream_t>(stream)));
}

int pf_gemm_dw_pairs(const void* dY, long long ldy, const void* X, long long ldx, float* G, long long ldg, int M,
                     int N, int K, const int* pairs, const int* pair_count, int* unit_stamp, int stamp_offset,
                     int stamp, void* stream) {
  if (!dY || !X || !G) return PF_ERR_INVALID;
  pf::DwGemm it{dY, ldy, X, ldx, G, ldg, M, N, K, pairs, pair_count, stamp_offset};
  return record(pf::gemm_dw_pairs(&it, 1, unit_stamp, stamp, static_cast<cudaStream_t>(stream)));
}

int pf_gemm_dw_dense(const void* dY, long long ldy, const void* X, long long ldx, float* G, long long ldg, int M,
                     int N, int K, int* unit_stamp, int stamp_offset, int stamp, void* stream) {
  if (!dY || !X || !G) return PF_ERR_INVALID;
  pf::DwGemm it{dY, ldy, X, ldx, G, ldg, M, N, K, nullptr, nullptr, stamp_offset};
  return record(pf::gemm_dw_dense(&it, 1, unit_stamp, stamp, static_cast<cudaStream_t>(stream)));
}

int pf_gemm_dw_rowpairs(const void* dY, long long ldy, const void* X, long long ldx, float* G, long long ldg, int M,
                        int N, int K, const int* entries, const int* entry_count, int* unit_stamp, int stamp_offset,
                        int stamp, void* stream) {
  if (!dY || !X || !G) return PF_ERR_INVALID;
  pf::DwGemm it{dY, ldy, X, ldx, G, ldg, M, N, K, entries, entry_count, stamp_offset};
  return record(pf::gemm_dw_rowpairs(&it, 1, unit_stamp, stamp, static_cast<cudaStream_t>(stream)));
}

int pf_gemm_swiglu(const void* h, long long ldh, const void* Wgu, long long ldw, void* gu, void* a, int T, int ffn,
                   int K, void* stream) {
  if (!h || !Wgu || !gu || !a || ffn % 128 != 0) return PF_ERR_INVALID;
  pf::GemmOut c{gu, 2LL * ffn};
  c.aux = a;
  c.ldaux = ffn;
  return record(pf::gemm_bf16_pair(pf::GemmOperand{h, ldh, false}, pf::GemmOperand{Wgu, ldw, false}, c, T, 2 * ffn,
                                   K, 1.0f, pf::EPI_SWIGLU, static_cast<cudaStream_t>(stream)));
}

int pf_gemm_dswiglu(const void* dY, long long ldy, const void* Wd, long long ldw, const void* gu, void* dgu, int T,
                    int ffn, int K, void* stream) {
  if (!dY || !Wd || !gu || !dgu || ffn % 128 != 0) return PF_ERR_INVALID;
  pf::GemmOut c{dgu, 2LL * ffn};
  c.residual = gu;
  c.ldr = 2LL * ffn;
  return record(pf::gemm_bf16_pair(pf::GemmOperand{dY, ldy, false}, pf::GemmOperand{Wd, ldw, true}, c, T, ffn, K,
                                   1.0f, pf::EPI_DSWIGLU, static_cast<cudaStream_t>(stream)));
}

int pf_gemm_gelu(const void* x, long long ldx, const void* W1, long long ldw, const void* bias, void* pre, void* act,
                 int T, int ffn, int K, void* stream) {
  if (!x || !W1 || !pre || !act || ffn % 32 != 0) return PF_ERR_INVALID;
  pf::GemmOut c{pre, ffn};
  c.aux = act;
  c.ldaux = ffn;
  c.bias = bias;
  return record(pf::gemm_bf16_pair(pf::GemmOperand{x, ldx, false}, pf::GemmOperand{W1, ldw, false}, c, T, ffn, K,
                                   1.0f, pf::EPI_GELU, static_cast<cudaStream_t>(stream)));
}

int pf_gemm_dgelu(const void* dY, long long ldy, const void* W2, long long ldw, const void* pre, void* dpre,
                  float* db, int T, int ffn, int K, void* stream) {
  if (!dY || !W2 || !pre || !dpre || ffn % 32 != 0) return PF_ERR_INVALID;
  pf::GemmOut c{dpre, ffn};
  c.residual = pre;
  c.ldr = ffn;
  c.colsum = db;
  return record(pf::gemm_bf16_pair(pf::GemmOperand{dY, ldy, false}, pf::GemmOperand{W2, ldw, true}, c, T, ffn, K,
                                   1.0f, pf::EPI_DGELU, static_cast<cudaStream_t>(stream)));
}

int pf_gemm_set_streamk(int mode) {
  if (mode < -1 || mode > 2) return PF_ERR_INVALID;
  pf::gemm_set_streamk(mode);
  return PF_OK;
}

int pf_device_sm_count(void) { return pf::num_sms(); }

const char* pf_device_last_error(void) { return g_last_error.c_str(); }

}  // extern "C"

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>

namespace pf {
namespace {
std::atomic<long long> g_launches{0};
}
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
// Per model family (set_pdl_default, from make_stage): on one B200 (bench.py, alternating runs)
// PDL moves the LLaMA-1B stable-freeze step by +0.3..0.6% (noise level) and slows its no-freeze
// step by 2-3%, so LLaMA stages keep it off; the ViT-L/32 step, thousands of small kernels,
// gains 7.5% (399k -> 429k tok/s), so ViT stages turn it on. PF_PDL=1 / PF_PDL=0 override both.
namespace {
std::atomic<int> g_pdl_default{0};
}
void set_pdl_default(bool on) { g_pdl_default.store(on ? 1 : 0, std::memory_order_relaxed); }
bool pdl_enabled() {
  static const int env = [] {
    const char* e = std::getenv("PF_PDL");
    return e ? (e[0] == '1' ? 1 : 0) : -1;
  }();
  return env >= 0 ? env == 1 : g_pdl_default.load(std::memory_order_relaxed) != 0;
}
long long launch_count() { return g_launches.load(std::memory_order_relaxed); }
bool trace_launches() {
  static const bool on = [] {
    const char* e = std::getenv("PF_TRACE_LAUNCH");
    return e && e[0] == '1';
  }();
  return on;
}
void trace_launch(const void* func, dim3 grid, cudaStream_t s) {
  const char* name = nullptr;
  if (cudaFuncGetName(&name, func) != cudaSuccess || !name) name = "?";
  std::fprintf(stderr, "[pf launch %lld] %s grid (%u,%u,%u) ...", launch_count(), name, grid.x, grid.y, grid.z);
  std::fflush(stderr);
  const auto t0 = std::chrono::steady_clock::now();
  const cudaError_t e = cudaStreamSynchronize(s);
  const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  std::fprintf(stderr, " %s %.3f ms\n", cudaGetErrorString(e), ms);
  std::fflush(stderr);
}
}  // namespace pf

extern "C" long long pf_device_launch_count(void) { return pf::launch_count(); }

#include <vector>

namespace pf {
namespace {
struct Probe {
  int kind = PROBE_OFF;
  std::vector<cudaEvent_t> ev;  // pairs
  std::size_t used = 0;         // events recorded
};
Probe& probe() {
  static Probe p;
  return p;
}
void probe_record(cudaStream_t s) {
  Probe& p = probe();
  if (p.used == p.ev.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    p.ev.push_back(e);
  }
  cudaEventRecord(p.ev[p.used++], s);
}
}  // namespace
int probe_kind() { return probe().kind; }
void probe_begin(cudaStream_t s) {
  if (probe().kind != PROBE_OFF) probe_record(s);
}
void probe_end(cudaStream_t s) {
  if (probe().kind != PROBE_OFF) probe_record(s);
}
}  // namespace pf

extern "C" int pf_probe_enable(int which) {
  if (which < 0 || which > 1) return PF_ERR_INVALID;
  pf::probe().kind = which;
  pf::probe().used = 0;
  return PF_OK;
}

extern "C" int pf_probe_read(int* launches, double* total_ms) {
  auto& p = pf::probe();
  double sum = 0.0;
  for (std::size_t i = 0; i + 1 < p.used; i += 2) {
    if (cudaEventSynchronize(p.ev[i + 1]) != cudaSuccess) return PF_ERR_CUDA;
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, p.ev[i], p.ev[i + 1]) != cudaSuccess) return PF_ERR_CUDA;
    sum += ms;
  }
  if (launches) *launches = static_cast<int>(p.used / 2);
  if (total_ms) *total_ms = sum;
  p.used = 0;
  return PF_OK;
}
