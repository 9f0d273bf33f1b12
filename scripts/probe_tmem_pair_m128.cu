// Probe: where does a cta_group::2 tcgen05.mma with M = 128 (64 A rows per
// CTA) put its accumulator rows in each CTA's TMEM?  (Needed for 128-row
// tail tiles in the CTA-pair expert GEMM; the PTX layout tables are not
// available offline.)  A[r][0] = r + 1, A[r][1] = 1; B[n][0] = 256,
// B[n][1] = n  =>  D[r][n] = 256 (r + 1) + n, decodable.  Both CTAs dump
// all 128 lanes x 256 columns; the host prints the (lane -> row) map.
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I include probe_tmem_pair_m128.cu
#include <cstdio>
#include <vector>

#include "../paper_2504_02263_b200/csrc/common.cuh"

using namespace msi;

template <int M>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) probe(float* out) {
  constexpr int AROWS = M / 2;   // A rows per CTA
  __shared__ __align__(1024) uint8_t sA[128 * 128];
  __shared__ __align__(1024) uint8_t sB[128 * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t s_tmem;
  const uint32_t rank = cluster_ctarank();
  const int tid = threadIdx.x;
  // fill A (AROWS x 64 K, SW128 K-major) and this CTA's B half (128 x 64)
  for (int i = tid; i < 128 * 64; i += blockDim.x) {
    const int row = i / 64, k = i % 64;
    const uint32_t off = row * 128 + ((((k * 2) >> 4) ^ (row & 7)) << 4) + ((k * 2) & 15);
    float a = 0.f, b = 0.f;
    const int r = row + (int)rank * AROWS;     // global A row
    const int n = row + (int)rank * 128;       // global B row (N index)
    if (row < AROWS) a = (k == 0) ? (float)(r + 1) : (k == 1 ? 1.f : 0.f);
    b = (k == 0) ? 256.f : (k == 1 ? (float)n : 0.f);
    *reinterpret_cast<__nv_bfloat16*>(sA + off) = __float2bfloat16(a);
    *reinterpret_cast<__nv_bfloat16*>(sB + off) = __float2bfloat16(b);
  }
  fence_proxy_async_shared();
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (tid < 32) tmem_alloc2<256>(&s_tmem);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  if (rank == 0 && tid == 0) {
    constexpr uint32_t idesc = umma_idesc_bf16(M, 256);
    mma_bf16_pair(tmem, umma_desc_sw128(sA), umma_desc_sw128(sB), idesc, 0);
    mma_commit_pair(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const int w = tid / 32, lane = tid % 32;
  for (int c = 0; c < 8; ++c) {
    uint32_t v[32];
    tmem_ld32(tmem + ((uint32_t)(w * 32) << 16) + c * 32, v);
    tmem_wait_ld();
    for (int j = 0; j < 32; ++j)
      out[((size_t)rank * 128 + w * 32 + lane) * 256 + c * 32 + j] = __uint_as_float(v[j]);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (tid < 32) tmem_dealloc2<256>(tmem);
}

template <int M>
void run() {
  float* d;
  cudaMalloc(&d, 2 * 128 * 256 * sizeof(float));
  cudaMemset(d, 0, 2 * 128 * 256 * sizeof(float));
  probe<M><<<2, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("M=%d: %s\n", M, cudaGetErrorString(e));
    return;
  }
  std::vector<float> h(2 * 128 * 256);
  cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
  printf("M=%d\n", M);
  for (int cta = 0; cta < 2; ++cta) {
    for (int lane = 0; lane < 128; ++lane) {
      // summarize the lane: decoded row, and column->n mapping of cols 0, 1, 127, 128, 255
      const float* L = &h[((size_t)cta * 128 + lane) * 256];
      int row = -1, bad = 0;
      int ns[5] = {0, 1, 127, 128, 255};
      char buf[256];
      int o = 0;
      for (int q = 0; q < 5; ++q) {
        const float v = L[ns[q]];
        const int iv = (int)v;
        const int r = iv / 256 - 1, n = iv % 256;
        if (v == 0.f) {
          o += snprintf(buf + o, sizeof(buf) - o, " c%d:0", ns[q]);
        } else {
          if (row < 0) row = r;
          else if (row != r) bad = 1;
          o += snprintf(buf + o, sizeof(buf) - o, " c%d:(r%d,n%d)", ns[q], r, n);
        }
      }
      if (lane % 8 == 0 || lane % 16 == 15) printf("cta%d lane%3d row%4d%s%s\n", cta, lane, row, bad ? " MIXED" : "", buf);
    }
  }
  cudaFree(d);
}

int main() {
  run<256>();
  run<128>();
  return 0;
}
