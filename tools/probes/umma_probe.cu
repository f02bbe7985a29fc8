// Development probe: cycles per tcgen05.mma (kind::f16, cta_group::1) for the operand shapes the
// attention kernels issue, back-to-back from one thread with precomputed descriptors (8 per loop).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2602_05754_b200/csrc/device \
//        tools/probes/umma_probe.cu -o tools/probes/umma_probe
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"

using namespace pf;

template <int V>
__global__ void probe(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) {
    tmem_alloc(&slot, 512);
    tmem_relinquish();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
    constexpr int N = (V == 1) ? 256 : 128;
    constexpr uint32_t id = V == 2 ? idesc_bf16_f32(128, N, false, true)
                          : V == 3 ? idesc_bf16_f32(128, N, true, true)
                                   : idesc_bf16_f32(128, N, false, false);
    uint64_t ad[8], bd[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      ad[k] = V == 3 ? sdesc_sw128(a + k * 2048, 16384, 1024) : sdesc_sw128(a + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
      bd[k] = (V == 2 || V == 3) ? sdesc_sw128(b + k * 2048, 16384, 1024)
                                 : sdesc_sw128(b + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
    }
    const long long t0 = clock64();
    for (int i = 0; i < iters; i += 8) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if constexpr (V == 2) umma_bf16_ts(tmem + 256, tmem + k * 8, bd[k], id, 1);
        else umma_bf16(tmem + (V == 4 ? (k & 1) * 128 : 0), ad[k], bd[k], id, 1);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

template <int V>
void run(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, 1024 * 8);
  cudaFuncSetAttribute(probe<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  const int iters = 4096, grid = 148;
  probe<V><<<grid, 128, 96 * 1024>>>(iters, d);
  probe<V><<<grid, 128, 96 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
  const int n = V == 1 ? 256 : 128;
  printf("%-44s %6.1f cycles/MMA = %6.0f flop/clk/SM  %s\n", name, mx / iters, 2.0 * 128 * n * 16 * iters / mx,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<0>("SS M128 N128 K-major (S = Q K^T)");
  run<1>("SS M128 N256 K-major");
  run<2>("TS M128 N128, B MN-major (O += P V)");
  run<3>("SS M128 N128 A,B MN-major (dQ = dS K)");
  run<4>("SS M128 N128, 2 accumulators");
  return 0;
}
