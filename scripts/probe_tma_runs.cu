// probe_tma_runs.cu -- does a 128B-swizzled TMA box land in shared memory
// swizzled by the *address* of each row (so a 128-row GEMM A tile can be
// assembled from row runs of any length at any row offset), or relative to the
// box start?  Loads the same 128 rows (a) as one 128-row box and (b) as a chain
// of power-of-two boxes (1, 2, 4, ... rows) at consecutive smem row offsets,
// and compares the two smem images byte for byte.  Also checks a run that
// starts at an odd global row.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o probe_tma_runs probe_tma_runs.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap m128, const __grid_constant__ CUtensorMap m64,
                      const __grid_constant__ CUtensorMap m32, const __grid_constant__ CUtensorMap m16,
                      const __grid_constant__ CUtensorMap m8, const __grid_constant__ CUtensorMap m4,
                      const __grid_constant__ CUtensorMap m2, const __grid_constant__ CUtensorMap m1,
                      int row0, int* mismatches) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* a = sm;                // full box
  uint8_t* b = sm + 128 * 128;    // pieces
  __shared__ __align__(8) uint64_t bar;
  const CUtensorMap* maps[8] = {&m128, &m64, &m32, &m16, &m8, &m4, &m2, &m1};
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(2 * 128 * 128) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(smem_u32(a)), "l"(maps[0]), "r"(0), "r"(row0), "r"(smem_u32(&bar)) : "memory");
    // pieces: 1 + 2 + 4 + 8 + 16 + 32 + 64 + 1 = 128 rows, consecutive
    const int sizes[8] = {1, 2, 4, 8, 16, 32, 64, 1};
    int r = 0;
    for (int i = 0; i < 8; ++i) {
      const int h = sizes[i];
      const int mi = h == 64 ? 1 : h == 32 ? 2 : h == 16 ? 3 : h == 8 ? 4 : h == 4 ? 5 : h == 2 ? 6 : 7;
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(smem_u32(b + r * 128)), "l"(maps[mi]), "r"(0), "r"(row0 + r), "r"(smem_u32(&bar)) : "memory");
      r += h;
    }
  }
  __syncthreads();
  asm volatile(
      "{\n.reg .pred P1;\nW: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(smem_u32(&bar)) : "memory");
  int bad = 0;
  for (int i = threadIdx.x; i < 128 * 128; i += blockDim.x) bad += a[i] != b[i];
  atomicAdd(mismatches, bad);
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int rows = 512, cols = 64;
  std::vector<uint16_t> h(rows * cols);
  for (int i = 0; i < rows * cols; ++i) h[i] = (uint16_t)(i * 2654435761u >> 7);
  void* d;
  CK(cudaMalloc(&d, h.size() * 2));
  CK(cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice));
  void* fp;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
  Enc enc = (Enc)fp;
  CUtensorMap m[8];
  const int hs[8] = {128, 64, 32, 16, 8, 4, 2, 1};
  for (int i = 0; i < 8; ++i) {
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows}, str[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)hs[i]}, es[2] = {1, 1};
    CUresult r = enc(&m[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) { printf("encode %d failed %d\n", hs[i], (int)r); return 1; }
  }
  int* mm;
  CK(cudaMalloc(&mm, 4));
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 128 * 128 + 1024));
  for (int row0 : {0, 1, 7, 13, 128, 255}) {
    CK(cudaMemset(mm, 0, 4));
    probe<<<1, 256, 2 * 128 * 128 + 1024>>>(m[0], m[1], m[2], m[3], m[4], m[5], m[6], m[7], row0, mm);
    CK(cudaDeviceSynchronize());
    int bad = 0;
    CK(cudaMemcpy(&bad, mm, 4, cudaMemcpyDeviceToHost));
    printf("{\"row0\": %d, \"mismatched_bytes\": %d, \"swizzle\": \"%s\"}\n", row0, bad,
           bad ? "relative to the box (runs must start on 8-row atoms)" : "by smem address (any row offset works)");
  }
  return 0;
}
