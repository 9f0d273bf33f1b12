// peer_store_probe.cu -- ceiling of SM-issued stores into a peer GPU's HBM over
// NVLink (the M2N dispatch/echo copy pattern), one direction and both
// directions at once.  Sweeps CTAs x threads x bytes-in-flight per thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peer_store_probe peer_store_probe.cu
//   ./peer_store_probe [MB]
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

template <int U>
__global__ void copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16) {
  // each warp moves 512 B chunks; U chunks in flight per warp (loads first, then stores)
  const size_t lane = threadIdx.x & 31;
  const size_t gw = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const size_t nw = (gridDim.x * (size_t)blockDim.x) >> 5;
  const size_t nchunk = n16 / 32;
  for (size_t c0 = gw * U; c0 < nchunk; c0 += nw * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (c0 + u < nchunk) v[u] = __ldg(src + (c0 + u) * 32 + lane);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (c0 + u < nchunk) dst[(c0 + u) * 32 + lane] = v[u];
  }
}


// TMA bulk variant: each CTA streams CH-byte chunks global -> smem (bulk load)
// -> peer (bulk store), NB chunks in flight per CTA, one elected thread.
template <int CH, int NB>
__global__ void bulk_kernel(const char* __restrict__ src, char* __restrict__ dst, size_t bytes) {
  extern __shared__ __align__(128) char buf[];
  __shared__ __align__(8) unsigned long long bar[NB];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < NB; ++i) {
    unsigned a = (unsigned)__cvta_generic_to_shared(&bar[i]);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a));
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const size_t nch = bytes / CH;
  unsigned phase[NB];
  for (int i = 0; i < NB; ++i) phase[i] = 0;
  int it = 0;
  for (size_t c = blockIdx.x; c < nch; c += gridDim.x, ++it) {
    const int b = it % NB;
    char* sb = buf + (size_t)b * CH;
    unsigned sa = (unsigned)__cvta_generic_to_shared(sb);
    unsigned ba = (unsigned)__cvta_generic_to_shared(&bar[b]);
    // the buffer's previous store must have read smem
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NB - 1) : "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ba), "r"(CH) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sa), "l"(src + c * CH), "r"(CH), "r"(ba) : "memory");
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }"
                 ::"r"(ba), "r"(phase[b]) : "memory");
    phase[b] ^= 1;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + c * CH), "r"(sa), "r"(CH) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

typedef void (*kfn)(const uint4*, uint4*, size_t);

int main(int argc, char** argv) {
  size_t mb = argc > 1 ? atoi(argv[1]) : 256;
  size_t bytes = mb << 20;
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) { printf("need 2 GPUs\n"); return 1; }
  void *s[2], *d[2];
  cudaStream_t st[2];
  cudaEvent_t e0[2], e1[2];
  for (int g = 0; g < 2; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaDeviceEnablePeerAccess(1 - g, 0));
    CK(cudaMalloc(&s[g], bytes));
    CK(cudaMalloc(&d[g], bytes));
    CK(cudaMemset(s[g], 1, bytes));
    CK(cudaStreamCreate(&st[g]));
    CK(cudaEventCreate(&e0[g]));
    CK(cudaEventCreate(&e1[g]));
  }
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  kfn ks[4] = {copy_kernel<2>, copy_kernel<4>, copy_kernel<8>, copy_kernel<16>};
  int us[4] = {2, 4, 8, 16};
  int grids[4] = {sms / 2, sms, 2 * sms, 4 * sms};
  int threads[3] = {256, 512, 1024};
  printf("{\"bytes\": %zu, \"sms\": %d}\n", bytes, sms);
  for (int bidir = 0; bidir < 2; ++bidir)
    for (int ki = 0; ki < 4; ++ki)
      for (int gi = 0; gi < 4; ++gi)
        for (int ti = 0; ti < 3; ++ti) {
          const int G = grids[gi], TH = threads[ti];
          if ((size_t)G * TH > 4 * 2048 * (size_t)sms) continue;
          cudaFuncAttributes fa;
          CK(cudaFuncGetAttributes(&fa, ks[ki]));
          if (TH > fa.maxThreadsPerBlock) continue;
          float best = 1e30f;
          for (int rep = 0; rep < 5; ++rep) {
            for (int g = 0; g <= bidir; ++g) {
              CK(cudaSetDevice(g));
              CK(cudaEventRecord(e0[g], st[g]));
              ks[ki]<<<G, TH, 0, st[g]>>>((const uint4*)s[g], (uint4*)d[1 - g], bytes / 16);
              CK(cudaEventRecord(e1[g], st[g]));
            }
            float ms = 0;
            for (int g = 0; g <= bidir; ++g) {
              CK(cudaSetDevice(g));
              CK(cudaEventSynchronize(e1[g]));
              float t;
              CK(cudaEventElapsedTime(&t, e0[g], e1[g]));
              ms = t > ms ? t : ms;
            }
            if (rep > 0 && ms < best) best = ms;
          }
          printf("{\"bidir\": %d, \"unroll\": %d, \"grid\": %d, \"threads\": %d, \"gbps_per_direction\": %.1f}\n",
                 bidir, us[ki], G, TH, bytes / (best * 1e-3) / 1e9);
        }
  // reference: cudaMemcpyPeerAsync (copy engines)
  for (int bidir = 0; bidir < 2; ++bidir) {
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      for (int g = 0; g <= bidir; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaEventRecord(e0[g], st[g]));
        CK(cudaMemcpyPeerAsync(d[1 - g], 1 - g, s[g], g, bytes, st[g]));
        CK(cudaEventRecord(e1[g], st[g]));
      }
      float ms = 0;
      for (int g = 0; g <= bidir; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaEventSynchronize(e1[g]));
        float t;
        CK(cudaEventElapsedTime(&t, e0[g], e1[g]));
        ms = t > ms ? t : ms;
      }
      if (rep > 0 && ms < best) best = ms;
    }
    printf("{\"bidir\": %d, \"memcpy_peer_gbps_per_direction\": %.1f}\n", bidir, bytes / (best * 1e-3) / 1e9);
  }
  // TMA bulk stores
  {
    struct V { void (*k)(const char*, char*, size_t); int ch, nb; const char* name; };
    V vs[] = {{bulk_kernel<4096, 8>, 4096, 8, "4K x8"}, {bulk_kernel<16384, 4>, 16384, 4, "16K x4"},
              {bulk_kernel<16384, 8>, 16384, 8, "16K x8"}, {bulk_kernel<32768, 4>, 32768, 4, "32K x4"},
              {bulk_kernel<12288, 8>, 12288, 8, "12K x8"}};
    for (auto& v : vs)
      for (int g = 0; g < 2; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaFuncSetAttribute(v.k, cudaFuncAttributeMaxDynamicSharedMemorySize, v.ch * v.nb));
      }
    for (int bidir = 0; bidir < 2; ++bidir)
      for (auto& v : vs)
        for (int mul = 1; mul <= 2; ++mul) {
          const int G = sms * mul;
          if ((size_t)v.ch * v.nb * mul > 200 * 1024) continue;
          float best = 1e30f;
          for (int rep = 0; rep < 5; ++rep) {
            for (int g = 0; g <= bidir; ++g) {
              CK(cudaSetDevice(g));
              CK(cudaEventRecord(e0[g], st[g]));
              v.k<<<G, 32, v.ch * v.nb, st[g]>>>((const char*)s[g], (char*)d[1 - g], bytes / v.ch * v.ch);
              CK(cudaGetLastError());
              CK(cudaEventRecord(e1[g], st[g]));
            }
            float ms = 0;
            for (int g = 0; g <= bidir; ++g) {
              CK(cudaSetDevice(g));
              CK(cudaEventSynchronize(e1[g]));
              float t;
              CK(cudaEventElapsedTime(&t, e0[g], e1[g]));
              ms = t > ms ? t : ms;
            }
            if (rep > 0 && ms < best) best = ms;
          }
          printf("{\"bidir\": %d, \"tma\": \"%s\", \"grid\": %d, \"gbps_per_direction\": %.1f}\n", bidir, v.name, G,
                 (bytes / v.ch * v.ch) / (best * 1e-3) / 1e9);
        }
  }
  return 0;
}
