// peer_load_probe.cu -- ceiling of SM-issued LOADS from a peer GPU's HBM over
// NVLink (a pull-style N2M combine) against SM stores into the peer (the push
// the dispatch / GEMM2 epilogue use): one direction, and both GPUs pulling
// from each other at once.  Each warp moves 512-B chunks with U chunks in
// flight.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peer_load_probe peer_load_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

template <int U>
__global__ void copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16) {
  const size_t lane = threadIdx.x & 31;
  const size_t gw = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const size_t nw = (gridDim.x * (size_t)blockDim.x) >> 5;
  const size_t nchunk = n16 / 32;
  for (size_t c0 = gw * U; c0 < nchunk; c0 += nw * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (c0 + u < nchunk) v[u] = __ldcg(src + (c0 + u) * 32 + lane);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (c0 + u < nchunk) dst[(c0 + u) * 32 + lane] = v[u];
  }
}

template <int U>
float run(int dev, const uint4* src, uint4* dst, size_t bytes, int grid, int block, cudaStream_t st) {
  CK(cudaSetDevice(dev));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  copy_kernel<U><<<grid, block, 0, st>>>(src, dst, bytes / 16);
  CK(cudaEventRecord(a, st));
  for (int i = 0; i < 5; ++i) copy_kernel<U><<<grid, block, 0, st>>>(src, dst, bytes / 16);
  CK(cudaEventRecord(b, st));
  CK(cudaEventSynchronize(b));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms / 5;
}

int main(int argc, char** argv) {
  const size_t MB = argc > 1 ? atoi(argv[1]) : 256;
  const size_t bytes = MB << 20;
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) { printf("{\"error\": \"needs 2 GPUs\"}\n"); return 0; }
  void *b0, *b1, *l0, *l1;
  CK(cudaSetDevice(0)); CK(cudaDeviceEnablePeerAccess(1, 0)); CK(cudaMalloc(&b0, bytes)); CK(cudaMalloc(&l0, bytes));
  CK(cudaMemset(b0, 1, bytes));
  CK(cudaSetDevice(1)); CK(cudaDeviceEnablePeerAccess(0, 0)); CK(cudaMalloc(&b1, bytes)); CK(cudaMalloc(&l1, bytes));
  CK(cudaMemset(b1, 2, bytes));
  cudaStream_t s0, s1;
  CK(cudaSetDevice(0)); CK(cudaStreamCreate(&s0));
  CK(cudaSetDevice(1)); CK(cudaStreamCreate(&s1));
  for (int grid : {148, 296, 592}) {
    for (int block : {256, 512}) {
      // pull: GPU 0 loads from GPU 1's buffer, stores locally
      float pull = run<8>(0, (const uint4*)b1, (uint4*)l0, bytes, grid, block, s0);
      // push: GPU 0 loads locally, stores into GPU 1
      float push = run<8>(0, (const uint4*)l0, (uint4*)b1, bytes, grid, block, s0);
      // both directions pulling at once
      CK(cudaSetDevice(0));
      cudaEvent_t a0, e0, a1, e1;
      CK(cudaEventCreate(&a0)); CK(cudaEventCreate(&e0));
      CK(cudaSetDevice(1)); CK(cudaEventCreate(&a1)); CK(cudaEventCreate(&e1));
      CK(cudaSetDevice(0)); CK(cudaEventRecord(a0, s0));
      for (int i = 0; i < 5; ++i) copy_kernel<8><<<grid, block, 0, s0>>>((const uint4*)b1, (uint4*)l0, bytes / 16);
      CK(cudaEventRecord(e0, s0));
      CK(cudaSetDevice(1)); CK(cudaEventRecord(a1, s1));
      for (int i = 0; i < 5; ++i) copy_kernel<8><<<grid, block, 0, s1>>>((const uint4*)b0, (uint4*)l1, bytes / 16);
      CK(cudaEventRecord(e1, s1));
      CK(cudaEventSynchronize(e1)); CK(cudaSetDevice(0)); CK(cudaEventSynchronize(e0));
      float m0 = 0, m1 = 0;
      CK(cudaEventElapsedTime(&m0, a0, e0));
      CK(cudaSetDevice(1)); CK(cudaEventElapsedTime(&m1, a1, e1));
      const double gb = bytes / 1e9;
      printf("{\"grid\": %d, \"block\": %d, \"pull_gbps\": %.1f, \"push_gbps\": %.1f, \"pull_bidir_gbps_per_dir\": %.1f}\n",
             grid, block, gb / (pull * 1e-3), gb / (push * 1e-3), gb / (((m0 + m1) / 2 / 5) * 1e-3));
    }
  }
  return 0;
}
