/* pipefreeze device C-ABI (libpf_device.so): hand-written sm_100a kernels and the
 * per-stage training step behind them.
 *
 * The reference (arXiv 2602.05754 `pipefreeze`) has no device layer: its stage
 * step is two CPU stand-ins, the duration model `sample_execution`
 * (proj/src/timing.cpp:58-65) and the masked-SGD numerics `run_masked_sgd`
 * (proj/src/sandbox.cpp:191-257). Each entry point below cites the reference
 * function whose semantics it realises on the device. All pointers are device
 * pointers unless named `host_*`; every call returns a PF_* status (pf_status.h)
 * and is asynchronous on the given stream.
 */
#ifndef PF_DEVICE_H
#define PF_DEVICE_H

#include <stddef.h>
#include <stdint.h>

#include "pf_status.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pf_ctx pf_ctx; /* opaque per-GPU stage context */

/* ------------------------------------------------------------------ kernels */

/* K1/K2/K3: C (op)= alpha * A . B^T with bf16 operands and fp32 TMEM accumulation.
 * A is logical [M,K]; a_mn_major=0: stored row-major [M][lda], 1: stored [K][lda].
 * B is logical [N,K]; b_mn_major=0: stored [N][ldb],       1: stored [K][ldb].
 * epilogue: 0 store bf16, 1 add into bf16 C, 2 fp32 unit-stamped accumulate
 * (requires unit_stamp, block_n=128), 3 store fp32. block_n in {128, 256}. */
int pf_gemm_bf16(const void* A, int a_mn_major, long long lda, const void* B, int b_mn_major,
                 long long ldb, void* C, long long ldc, int M, int N, int K, float alpha,
                 int epilogue, int block_n, int* unit_stamp, int stamp, void* stream);

/* K3: masked weight gradient G[M,N] += alpha * A . B^T over the 128x128 units
 * listed in unit_list[0..*unit_count) (unit id = row_block * ceil(N/128) + col_block).
 * First touch of a unit in step `stamp` stores, later touches accumulate
 * (G = sum_m U_m . g_m, reference proj/src/sandbox.cpp:232-249). */
int pf_gemm_dw_units(const void* A, int a_mn_major, long long lda, const void* B, int b_mn_major,
                     long long ldb, float* G, long long ldg, int M, int N, int K, float alpha,
                     const int* unit_list, const int* unit_count, int max_units,
                     int* unit_stamp, int stamp_offset, int stamp, void* stream);

int pf_device_sm_count(void);
const char* pf_device_last_error(void);

#ifdef __cplusplus
}
#endif

#endif
