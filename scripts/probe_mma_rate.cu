// Probe: tcgen05.mma kind::f16 issue rate by shape, one CTA (or CTA pair)
// per SM issuing back-to-back MMAs from shared memory (no loads, no
// epilogue).  Question it settles: does an M = 64
// cta_group::1 MMA run at the per-SM rate of an M = 128 one, i.e. would
// 64-row "quarter" tail units of the expert GEMM save MMA time?
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 probe_mma_rate.cu -o probe_mma_rate
#include <cstdio>

#include "../paper_2504_02263_b200/csrc/common.cuh"

using namespace msi;

constexpr int kIters = 16384;  // MMAs (K = 16 each) per CTA or pair

template <int M, int N, int CG>
__global__ void __launch_bounds__(128, 1) mma_rate(int dummy) {
  extern __shared__ uint8_t dsm[];
  uint8_t* sA = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
  uint8_t* sB = sA + 128 * 128;
  constexpr int kA = 128 * 128, kB = 256 * 128;
  __shared__ uint64_t bar;
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x;
  for (int i = tid; i < kA / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sA)[i] = 0x3f803f80u * dummy;
  for (int i = tid; i < kB / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sB)[i] = 0x3f803f80u * dummy;
  fence_proxy_async_shared();
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (tid < 32) {
    if constexpr (CG == 2) tmem_alloc2<256>(&s_tmem);
    else tmem_alloc<256>(&s_tmem);
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  const bool issuer = tid == 0 && (CG == 1 || cluster_ctarank() == 0);
  if (issuer) {
    constexpr uint32_t idesc = umma_idesc_bf16(M, N);
    const uint64_t ad = umma_desc_sw128(sA), bd = umma_desc_sw128(sB);
    for (int i = 0; i < kIters; ++i) {
      // K = 16 steps through the 64-wide SW128 atom (+32 B per step), as the GEMM does
      const uint64_t k = (uint64_t)((i & 3) * 2);
      if constexpr (CG == 2) mma_bf16_pair(tmem, ad + k, bd + k, idesc, i > 0);
      else mma_bf16(tmem, ad + k, bd + k, idesc, i > 0);
    }
    if constexpr (CG == 2) mma_commit_pair(&bar);
    else mma_commit(&bar);
  }
  if (CG == 1 || cluster_ctarank() == 0) mbar_wait(&bar, 0);
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync();
  tc_fence_after();
  if (tid < 32) {
    if constexpr (CG == 2) tmem_dealloc2<256>(tmem);
    else tmem_dealloc<256>(tmem);
  }
}

template <int M, int N, int CG>
void run(int sms) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int grid = sms - (sms % 2);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const int smem = 128 * 128 + 256 * 128 + 1024;
  cudaFuncSetAttribute(mma_rate<M, N, CG>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cfg.dynamicSmemBytes = smem;
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a);
    cudaLaunchKernelEx(&cfg, mma_rate<M, N, CG>, 1);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    if (e != cudaSuccess) {
      printf("M=%d N=%d cg=%d: %s\n", M, N, CG, cudaGetErrorString(e));
      return;
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (rep > 0 && ms < best) best = ms;
  }
  const double issuers = CG == 2 ? grid / 2 : grid;
  const double flop = issuers * kIters * 2.0 * M * N * 16;
  printf("{\"M\": %d, \"N\": %d, \"cta_group\": %d, \"ctas\": %d, \"ms\": %.4f, \"tflops\": %.1f, "
         "\"ns_per_mma\": %.2f}\n", M, N, CG, grid, best, flop / best / 1e9, best * 1e6 / kIters);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<128, 256, 1>(sms);
  run<64, 256, 1>(sms);
  run<128, 128, 1>(sms);
  run<64, 128, 1>(sms);
  run<256, 256, 2>(sms);
  run<128, 256, 2>(sms);
  return 0;
}
