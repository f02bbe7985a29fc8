// Internal (C++) declarations shared by the device translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "pf_status.h"

namespace pf {

enum GemmEpilogue : int {
  EPI_STORE_BF16 = 0,  // C = bf16(alpha * acc)
  EPI_ADD_BF16 = 1,    // C = bf16(C + alpha * acc)
  EPI_ACC_F32 = 2,     // fp32 C; first touch of a 128x128 unit in this step stores, later add
  EPI_STORE_F32 = 3,   // C = alpha * acc (fp32)
  EPI_SWIGLU = 4,      // CTA pair only: C = bf16(gate|up), aux = silu(gate) * up (interleaved 128-blocks)
  EPI_DSWIGLU = 5,     // CTA pair only: acc = d(act) [M][ffn]; residual = gu; C = d(gate|up), same layout as gu
  EPI_GELU = 6,        // CTA pair only: C = pre = bf16(acc + bias), aux = gelu(pre)      (ViT fc1)
  EPI_DGELU = 7,       // CTA pair only: acc = d(act); residual = pre; C = d(act) * gelu'(pre) (ViT fc2 dX)
  EPI_ROPE = 8,        // CTA pair only: C = qkv with rotate-half RoPE on the q and k heads (head_dim 64)
};

struct GemmOperand {
  const void* ptr;    // bf16
  long long ld;       // row stride in elements of the stored matrix
  bool mn_major;      // false: stored [rows][K]; true: stored [K][rows]
};

struct GemmOut {
  void* ptr;
  long long ld;
  int* unit_stamp = nullptr;  // EPI_ACC_F32 only
  int stamp_offset = 0;
  int stamp = 0;
  const void* residual = nullptr;  // EPI_ADD_BF16 on the CTA-pair kernel: C = R + acc (R may differ from C)
  long long ldr = 0;
  void* aux = nullptr;  // EPI_SWIGLU: [M][N/2] bf16 activation
  long long ldaux = 0;
  const void* bias = nullptr;  // CTA-pair EPI_STORE_BF16 / EPI_ADD_BF16: + bias[col] (bf16 [N])
  float* colsum = nullptr;     // CTA-pair EPI_DGELU: += column sums of the bf16 output (a bias gradient)
  const void* rope = nullptr;  // CTA-pair EPI_ROPE: float2 (cos, sin) table [seq][rope_hd / 2]
  int rope_hd = 64;            // EPI_ROPE: head_dim, 64 or 128
  int rope_seq = 0;            // EPI_ROPE: positions per sequence (row t is position t % seq)
  int rope_cols = 0;           // EPI_ROPE: columns [0, rope_cols) are q and k heads (rotated)
};

int gemm_bf16(const GemmOperand& A, const GemmOperand& B, const GemmOut& C, int M, int N, int K,
              float alpha, int epi, int block_n, cudaStream_t stream);

// Masked weight-gradient GEMM over a device-resident list of 128x128 units
// (dY and X MN-major, alpha = 1; one matrix of gemm_dw_units).
int gemm_bf16_units(const GemmOperand& A, const GemmOperand& B, const GemmOut& C, int M, int N,
                    int K, float alpha, const int* unit_list, const int* unit_count,
                    int max_units, cudaStream_t stream);

// K3, batched: the masked dW of many matrices (every matrix of a microbatch) in one
// persistent launch. One work item per matrix: G (+)= dY^T . X over its unfrozen units.
constexpr int kMaxDwProblems = 96;  // matrices per launch (kernel parameter space <= 32 KB)
struct DwGemm {
  const void* dy;    // bf16 [K][M]: output-feature gradient (MN-major A)
  long long ldy;
  const void* x;     // bf16 [K][N]: layer input (MN-major B)
  long long ldx;
  float* C;          // fp32 gradient of the matrix [M][N]
  long long ldc;
  int M, N, K;
  const int* list;   // device work list of this matrix (K5 unit list / K5p pair list)
  const int* count;  // device: entry count
  int stamp_offset;  // first unit id of the matrix in the stage
};
// 1-CTA 128 x 128 tiles over K5 unit lists (gemm.cu) -- the default
int gemm_dw_units(const DwGemm* items, int n, int* unit_stamp, int stamp, cudaStream_t stream);
// CTA-pair 256 x 128 tiles over K5p pair lists (gemm_dw.cu; PF_DW_PAIR=1)
int gemm_dw_pairs(const DwGemm* items, int n, int* unit_stamp, int stamp, cudaStream_t stream);
// 1-CTA 128 x 256 tiles over K5r row-pair lists: two units of one row per MMA (gemm_dw_rows.cu)
int gemm_dw_rowpairs(const DwGemm* items, int n, int* unit_stamp, int stamp, cudaStream_t stream);
// Every unit of every matrix (a cell with no frozen unit): 256 x 256 CTA-pair tiles, list-free
// (gemm_dw.cu); same unit-stamp contract.
int gemm_dw_dense(const DwGemm* items, int n, int* unit_stamp, int stamp, cudaStream_t stream);

// K1/K2 on a CTA pair (cta_group::2, 256 x 256 tiles); A must be K-major.
int gemm_bf16_pair(const GemmOperand& A, const GemmOperand& B, const GemmOut& C, int M, int N, int K, float alpha,
                   int epi, cudaStream_t stream);

// Stream-K for the CTA-pair kernel: -1 auto, 0 off (default, or PF_GEMM_STREAMK), 1 force.
void gemm_set_streamk(int mode);

int num_sms();

// In-step probe of one kernel (bench.py roofline: average duration of the dominant
// kernel measured inside the timed steps, on the launching stream).
enum ProbeKind : int { PROBE_OFF = 0, PROBE_GATE_UP_GEMM = 1 };
int probe_kind();
void probe_begin(cudaStream_t s);  // no-op unless the probe is enabled
void probe_end(cudaStream_t s);

// Programmatic dependent launch (PDL): every kernel of this library is launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, waits (griddepcontrol.wait) for the
// previous kernel's completion and memory before touching global memory, and lets the next
// kernel launch early (griddepcontrol.launch_dependents), so a kernel's launch and prologue
// overlap its predecessor's tail. Default per model family (set_pdl_default: ViT on, LLaMA
// off; measured: capi_kernels.cu), PF_PDL=0|1 overrides. The kernels always execute
// griddepcontrol.wait / launch_dependents (no-ops without the attribute).
bool pdl_enabled();
void set_pdl_default(bool on);

// PF_TRACE_LAUNCH=1 (debugging a hung step): every launch_k prints the kernel's name and grid to
// stderr, synchronises its stream and prints the elapsed time, so the last line names a kernel
// that never finished.
bool trace_launches();
void trace_launch(const void* func, dim3 grid, cudaStream_t s);

// Number of kernels this library has launched (evidence for bench.py gpu_launches).
void count_launch();
long long launch_count();

}  // namespace pf
