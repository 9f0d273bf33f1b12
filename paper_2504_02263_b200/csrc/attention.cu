// attention.cu -- the attention stage's decode kernels.
//
// The reference has no attention kernel: it models the stage as
// T_a = k1*b_a + k2 with the KV-cache read 2*b*s*h*bytes/g dominating
// ("KV cache access time is nearly
// proportional to b_a*s").  This file makes that stage real on B200:
//
//  * rope_append_kernel   -- RoPE (rotate-half) on the new token's q and k,
//                            then k/v appended into the paged cache.
//  * decode_attn_kernel   -- GQA decode attention over the paged cache.  It is
//    HBM-bound (every cached K/V byte is read once per step), so it is built
//    around the memory system: one CTA per (sequence, KV head[, KV split]);
//    a producer warp streams each (page, KV head) K and V tile (64 tokens x
//    128 dims = 16 KB, contiguous in the cache) with one 3-D TMA load each,
//    128B-swizzled, through a 3-stage mbarrier ring; four consumer warps take
//    16 tokens of every page each.  The G = n_heads/n_kv query heads that
//    share the KV head form the M rows of m16n8k16 bf16 MMAs (S = Q K^T, then
//    O += P V with P re-packed from the S accumulators in registers), with an
//    online (flash) softmax per warp and a 4-warp merge through shared memory.
//    The tensor work is ~8 FLOP per cached byte, far below the MMA roofline,
//    so mma.sync is sufficient here; the bytes are what matter.
//  * attn_split_combine_kernel -- merges split-KV partials when the batch is
//    too small to fill 148 SMs with one CTA per (sequence, KV head).
#include <algorithm>
#include <cmath>

#include "common.cuh"

namespace msi {

int num_sms();

namespace {

constexpr int kPage = MSI_KV_PAGE;          // tokens per page
constexpr int kD = MSI_HEAD_DIM;            // head dim
constexpr int kStages = 3;
constexpr int kTileBytes = kPage * kD * 2;  // 16 KB: one (page, KV head) K or V tile
constexpr int kCWarps = 4;                  // consumer warps (16 tokens of a page each)
constexpr int kThreads = (kCWarps + 1) * 32;
constexpr int kSmem = 1024 + kStages * 2 * kTileBytes + 2 * kStages * 8;

static_assert(kPage == kCWarps * 16, "one 16-token slice per consumer warp");
static_assert(kCWarps * 16 * kD * 4 + kCWarps * 16 * 8 <= kStages * 2 * kTileBytes,
              "merge scratch reuses the stage ring");

// 128B swizzle of a byte offset inside a 1024B-aligned tile (what TMA's
// SWIZZLE_128B applies on the way in): 16B chunk ^= (128B line index mod 8).
__device__ __forceinline__ uint32_t swz(uint32_t o) { return o ^ (((o >> 7) & 7u) << 4); }

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

struct AttnArgs {
  const __nv_bfloat16* q;  // [T][n_heads][128]
  const int* bt;           // [T][max_pages]
  const int* lens;         // [T]
  __nv_bfloat16* out;      // [T][n_heads][128]
  float* part_o;           // [T][n_heads][splits][128]   (splits > 1)
  float* part_ml;          // [T][n_heads][splits][2]
  int max_pages, T, n_heads, n_kv, G, splits, pps;
  float scale_log2;
};

__global__ void __launch_bounds__(kThreads, 2)
    decode_attn_kernel(const __grid_constant__ CUtensorMap tk, const __grid_constant__ CUtensorMap tv,
                       const __grid_constant__ CUtensorMap tk16, const __grid_constant__ CUtensorMap tv16,
                       const AttnArgs a) {
  extern __shared__ uint8_t smem_raw[];
  pdl_trigger();
  pdl_wait();
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * 2 * kTileBytes);
  uint64_t* empty = full + kStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  int id = blockIdx.x;
  const int split = id % a.splits;
  id /= a.splits;
  const int kvh = id % a.n_kv;
  const int seq = id / a.n_kv;
  const int len = a.lens[seq];
  const int npg = (len + kPage - 1) / kPage;
  const int pps = (npg + a.splits - 1) / a.splits;  // this sequence's pages per split
  const int p0 = split * pps;
  const int np = max(0, min(npg - p0, pps));

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kCWarps) {  // ---- producer: one elected thread streams K/V tiles
    if (lane == 0) {
      tma_prefetch(&tk);
      tma_prefetch(&tv);
      tma_prefetch(&tk16);
      tma_prefetch(&tv16);
      const int* btr = a.bt + (size_t)seq * a.max_pages + p0;
      for (int i = 0; i < np; ++i) {
        const int s = i % kStages;
        if (i >= kStages) mbar_wait(&empty[s], ((i / kStages) - 1) & 1);
        const int row = (btr[i] * a.n_kv + kvh) * kPage;
        const int valid = len - (p0 + i) * kPage;  // rows of this page in use (>= 1)
        if (valid >= kPage) {
          mbar_expect_tx(&full[s], 2 * kTileBytes);
          tma_load_3d(smem + s * 2 * kTileBytes, &tk, 0, 0, row, &full[s]);
          tma_load_3d(smem + s * 2 * kTileBytes + kTileBytes, &tv, 0, 0, row, &full[s]);
        } else {  // a sequence's last, partial page: only the 16-row groups in use
          const int nq = (valid + 15) / 16;
          mbar_expect_tx(&full[s], 2 * nq * (kTileBytes / 4));
          for (int q = 0; q < nq; ++q) {
            tma_load_3d(smem + s * 2 * kTileBytes + q * (kTileBytes / 4), &tk16, 0, 0, row + 16 * q, &full[s]);
            tma_load_3d(smem + s * 2 * kTileBytes + kTileBytes + q * (kTileBytes / 4), &tv16, 0, 0, row + 16 * q,
                        &full[s]);
          }
        }
      }
    }
    return;
  }

  // ---- consumers
  const int g = lane >> 2, c = lane & 3;
  const int G = a.G;
  const int h0 = kvh * G;
  uint32_t qa[8][4];
  {
    const uint32_t* q32 = reinterpret_cast<const uint32_t*>(a.q + ((size_t)seq * a.n_heads + h0) * kD);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const int col = kk * 16 + 2 * c;
      qa[kk][0] = g < G ? q32[(g * kD + col) >> 1] : 0u;
      qa[kk][1] = g + 8 < G ? q32[((g + 8) * kD + col) >> 1] : 0u;
      qa[kk][2] = g < G ? q32[(g * kD + col + 8) >> 1] : 0u;
      qa[kk][3] = g + 8 < G ? q32[((g + 8) * kD + col + 8) >> 1] : 0u;
    }
  }
  float o[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  const int lj = lane >> 3, lr = lane & 7;

  for (int i = 0; i < np; ++i) {
    const int s = i % kStages;
    mbar_wait(&full[s], (i / kStages) & 1);
    const int tok0 = (p0 + i) * kPage + warp * 16;
    if (tok0 < len) {
      const uint32_t kb = smem_u32(smem + s * 2 * kTileBytes);
      const uint32_t vb = kb + kTileBytes;
      const int nvalid = len - tok0;  // >= 1
      if (nvalid < 16) {
        // V rows past the end hold stale cache bytes (possibly NaN patterns):
        // P is 0 there, but 0 * NaN is not, so clear them before P V.
        uint8_t* vrows = smem + s * 2 * kTileBytes + kTileBytes;
        for (int e = lane; e < (16 - nvalid) * 16; e += 32) {
          const int r = warp * 16 + nvalid + e / 16;
          *reinterpret_cast<uint4*>(vrows + swz(r * 256 + (e % 16) * 16)) = make_uint4(0, 0, 0, 0);
        }
        __syncwarp();
      }
      float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        uint32_t b0, b1, b2, b3;
        const int trow = warp * 16 + lr + ((lj & 2) ? 8 : 0);
        const int dim = kk * 16 + ((lj & 1) ? 8 : 0);
        ldsm_x4(kb + swz(trow * 256 + dim * 2), b0, b1, b2, b3);
        mma16816(sc[0], qa[kk], b0, b1);
        mma16816(sc[1], qa[kk], b2, b3);
      }
#pragma unroll
      for (int n = 0; n < 2; ++n)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int tok = tok0 + n * 8 + 2 * c + (e & 1);
          sc[n][e] = tok < len ? sc[n][e] * a.scale_log2 : -INFINITY;
        }
      float mx0 = fmaxf(fmaxf(sc[0][0], sc[0][1]), fmaxf(sc[1][0], sc[1][1]));
      float mx1 = fmaxf(fmaxf(sc[0][2], sc[0][3]), fmaxf(sc[1][2], sc[1][3]));
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
      const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);  // finite: token tok0 is valid
      const float al0 = exp2f(m0 - mn0), al1 = exp2f(m1 - mn1);
      m0 = mn0;
      m1 = mn1;
#pragma unroll
      for (int n = 0; n < 2; ++n) {
        sc[n][0] = exp2f(sc[n][0] - mn0);
        sc[n][1] = exp2f(sc[n][1] - mn0);
        sc[n][2] = exp2f(sc[n][2] - mn1);
        sc[n][3] = exp2f(sc[n][3] - mn1);
      }
      l0 = l0 * al0 + (sc[0][0] + sc[0][1] + sc[1][0] + sc[1][1]);
      l1 = l1 * al1 + (sc[0][2] + sc[0][3] + sc[1][2] + sc[1][3]);
#pragma unroll
      for (int nt = 0; nt < 16; ++nt) {
        o[nt][0] *= al0;
        o[nt][1] *= al0;
        o[nt][2] *= al1;
        o[nt][3] *= al1;
      }
      const uint32_t pa[4] = {pack_bf16x2(sc[0][0], sc[0][1]), pack_bf16x2(sc[0][2], sc[0][3]),
                              pack_bf16x2(sc[1][0], sc[1][1]), pack_bf16x2(sc[1][2], sc[1][3])};
#pragma unroll
      for (int dp = 0; dp < 8; ++dp) {
        uint32_t b0, b1, b2, b3;
        const int trow = warp * 16 + lr + ((lj & 1) ? 8 : 0);
        const int dim = dp * 16 + ((lj & 2) ? 8 : 0);
        ldsm_x4_t(vb + swz(trow * 256 + dim * 2), b0, b1, b2, b3);
        mma16816(o[2 * dp], pa, b0, b1);
        mma16816(o[2 * dp + 1], pa, b2, b3);
      }
      if (nvalid < 16) fence_proxy_async_shared();  // generic writes before the next TMA fill
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);

  // ---- merge the four warps' (m, l, O) through the (drained) stage ring
  named_bar(1, kCWarps * 32);
  float* so = reinterpret_cast<float*>(smem);       // [warp][16 rows][128]
  float* sml = so + kCWarps * 16 * kD;               // [warp][16 rows][2]
#pragma unroll
  for (int nt = 0; nt < 16; ++nt) {
    const int d = nt * 8 + 2 * c;
    if (g < G) *reinterpret_cast<float2*>(&so[(warp * 16 + g) * kD + d]) = make_float2(o[nt][0], o[nt][1]);
    if (g + 8 < G)
      *reinterpret_cast<float2*>(&so[(warp * 16 + g + 8) * kD + d]) = make_float2(o[nt][2], o[nt][3]);
  }
  if (c == 0) {
    if (g < G) {
      sml[(warp * 16 + g) * 2] = m0;
      sml[(warp * 16 + g) * 2 + 1] = l0;
    }
    if (g + 8 < G) {
      sml[(warp * 16 + g + 8) * 2] = m1;
      sml[(warp * 16 + g + 8) * 2 + 1] = l1;
    }
  }
  named_bar(1, kCWarps * 32);
  const int d = threadIdx.x;  // 0..127
  for (int r = 0; r < G; ++r) {
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kCWarps; ++w) M = fmaxf(M, sml[(w * 16 + r) * 2]);
    float L = 0.f, O = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int w = 0; w < kCWarps; ++w) {
        const float f = exp2f(sml[(w * 16 + r) * 2] - M);
        L += sml[(w * 16 + r) * 2 + 1] * f;
        O += so[(w * 16 + r) * kD + d] * f;
      }
    }
    const size_t hrow = (size_t)seq * a.n_heads + h0 + r;
    if (a.splits == 1) {
      a.out[hrow * kD + d] = __float2bfloat16_rn(L > 0.f ? O / L : 0.f);
    } else {
      const size_t prow = hrow * a.splits + split;
      a.part_o[prow * kD + d] = O;
      if (d == 0) {
        a.part_ml[prow * 2] = M;
        a.part_ml[prow * 2 + 1] = L;
      }
    }
  }
}

__global__ void attn_split_combine_kernel(const float* __restrict__ part_o, const float* __restrict__ part_ml,
                                          int splits, __nv_bfloat16* __restrict__ out) {
  const size_t hrow = blockIdx.x;
  const int d = threadIdx.x;
  pdl_trigger();
  pdl_wait();
  const float* ml = part_ml + hrow * splits * 2;
  float M = -INFINITY;
  for (int s = 0; s < splits; ++s) M = fmaxf(M, ml[2 * s]);
  float L = 0.f, O = 0.f;
  if (M != -INFINITY)
    for (int s = 0; s < splits; ++s) {
      const float f = exp2f(ml[2 * s] - M);
      L += ml[2 * s + 1] * f;
      O += part_o[(hrow * splits + s) * kD + d] * f;
    }
  out[hrow * kD + d] = __float2bfloat16_rn(L > 0.f ? O / L : 0.f);
}

// One CTA per token: the token's 64 (cos, sin) pairs of pos * theta^(-2i/128)
// once into shared memory, then q (n_heads) and k (n_kv) rotated 8 pairs per
// thread with 16 B loads/stores (pairs (i, i+64)); q to q_out, k and v into
// the cache slot.
__global__ void rope_append_kernel(const __nv_bfloat16* __restrict__ qkv, int64_t ld, const int* __restrict__ pos,
                                   int n_heads, int n_kv, const __grid_constant__ RopeInv rope,
                                   const int* __restrict__ bt, int max_pages,
                                   __nv_bfloat16* __restrict__ kc, __nv_bfloat16* __restrict__ vc,
                                   __nv_bfloat16* __restrict__ q_out) {
  __shared__ float s_cos[kD / 2], s_sin[kD / 2];
  const int t = blockIdx.x;
  pdl_trigger();
  pdl_wait();
  const int p = pos[t];
  if (threadIdx.x < kD / 2) {
    const int i = threadIdx.x;
    sincosf((float)p * rope.v[i], &s_sin[i], &s_cos[i]);
  }
  __syncthreads();
  const int page = bt[(size_t)t * max_pages + p / kPage];
  const int prow = p % kPage;
  const __nv_bfloat16* src = qkv + (size_t)t * ld;
  const int nrot = (n_heads + n_kv) * 8;  // (head, 8-pair chunk)
  for (int w = threadIdx.x; w < nrot; w += blockDim.x) {
    const int head = w >> 3, c = w & 7;
    const __nv_bfloat16* hs = src + (size_t)head * kD;
    const uint4 lo4 = *reinterpret_cast<const uint4*>(hs + 8 * c);
    const uint4 hi4 = *reinterpret_cast<const uint4*>(hs + 64 + 8 * c);
    const uint32_t lo[4] = {lo4.x, lo4.y, lo4.z, lo4.w}, hi[4] = {hi4.x, hi4.y, hi4.z, hi4.w};
    uint32_t ro[4], rh[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i0 = 8 * c + 2 * j;
      const float x0a = bf16lo(lo[j]), x0b = bf16hi(lo[j]);
      const float x1a = bf16lo(hi[j]), x1b = bf16hi(hi[j]);
      const float ca = s_cos[i0], sa = s_sin[i0], cb = s_cos[i0 + 1], sb = s_sin[i0 + 1];
      ro[j] = pack_bf16x2(x0a * ca - x1a * sa, x0b * cb - x1b * sb);
      rh[j] = pack_bf16x2(x1a * ca + x0a * sa, x1b * cb + x0b * sb);
    }
    __nv_bfloat16* dst = head < n_heads ? q_out + ((size_t)t * n_heads + head) * kD
                                        : kc + (((size_t)page * n_kv + (head - n_heads)) * kPage + prow) * kD;
    *reinterpret_cast<uint4*>(dst + 8 * c) = make_uint4(ro[0], ro[1], ro[2], ro[3]);
    *reinterpret_cast<uint4*>(dst + 64 + 8 * c) = make_uint4(rh[0], rh[1], rh[2], rh[3]);
  }
  // v: n_kv heads x 128 dims, 16B vectors
  const uint4* vs = reinterpret_cast<const uint4*>(src + (size_t)(n_heads + n_kv) * kD);
  for (int w = threadIdx.x; w < n_kv * kD / 8; w += blockDim.x) {
    const int head = w / (kD / 8), v = w % (kD / 8);
    reinterpret_cast<uint4*>(vc + (((size_t)page * n_kv + head) * kPage + prow) * kD)[v] = vs[w];
  }
}

typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                      CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                      CUtensorMapFloatOOBfill);

// Cache tile map: the cache viewed as [rows][2 halves][64 dims] (rows =
// num_pages * n_kv * 64), box = one (page, KV head) tile, SWIZZLE_128B.
int kv_tmap(CUtensorMap* m, const void* base, uint64_t rows, uint32_t box_rows) {
  static PFN_encodeTiled_t enc = nullptr;
  if (!enc) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      set_error("cuTensorMapEncodeTiled unavailable");
      return MSI_EDRIVER;
    }
    enc = reinterpret_cast<PFN_encodeTiled_t>(p);
  }
  cuuint64_t dims[3] = {64, 2, rows};
  cuuint64_t strides[2] = {128, 256};
  cuuint32_t box[3] = {64, 2, box_rows};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (kv cache) failed (%d): rows=%llu", (int)r, (unsigned long long)rows);
    return MSI_EDRIVER;
  }
  return 0;
}

// Split-KV factor: one CTA per (sequence, KV head) when that fills the
// resident CTA slots (2 per SM), else split every sequence's pages
// evenly into `splits` parts (per sequence, so ragged lengths stay balanced).
void choose_splits(int T, int n_kv, int max_pages, int* splits, int* pps) {
  const long items = (long)T * n_kv;
  const long want = 2L * num_sms();  // (4x measured slower at T = 64: the combine pass costs more)
  int s = 1;
  if (items < want && max_pages > 1) s = (int)std::min<long>({(long)max_pages, 8L, (want + items - 1) / items});
  *splits = std::max(s, 1);
  *pps = (max_pages + *splits - 1) / *splits;  // upper bound (the kernel splits each sequence by its own length)
}

}  // namespace
}  // namespace msi

using namespace msi;

extern "C" int msi_rope_append(const void* qkv, int64_t qkv_ld, const int32_t* pos, int T, int n_heads, int n_kv,
                               float theta, const int32_t* block_table, int max_pages, void* k_cache,
                               void* v_cache, int64_t num_pages, void* q_out, void* stream) {
  MSI_REQUIRE(T >= 0 && n_kv > 0 && n_heads > 0 && n_heads % n_kv == 0, "rope_append: bad head counts");
  MSI_REQUIRE(qkv_ld >= (int64_t)(n_heads + 2 * n_kv) * MSI_HEAD_DIM && qkv_ld % 8 == 0,
              "rope_append: qkv_ld too small or not a multiple of 8");
  MSI_REQUIRE(theta > 0.f && max_pages > 0 && num_pages > 0, "rope_append: bad theta / page counts");
  MSI_REQUIRE(qkv && pos && block_table && k_cache && v_cache && q_out, "rope_append: null pointer");
  if (T == 0) return 0;
  MSI_CUDA(launch_k(rope_append_kernel, dim3(T), dim3(128), 0, (cudaStream_t)stream, (const __nv_bfloat16*)qkv,
                    (int64_t)qkv_ld, pos, n_heads, n_kv, rope_inv_table(theta), block_table, max_pages, (__nv_bfloat16*)k_cache,
                    (__nv_bfloat16*)v_cache, (__nv_bfloat16*)q_out));
  return check_launch("rope_append_kernel");
}

extern "C" size_t msi_decode_attention_workspace(int T, int n_heads, int n_kv, int max_pages) {
  if (T <= 0 || n_kv <= 0 || max_pages <= 0) return 0;
  int splits, pps;
  choose_splits(T, n_kv, max_pages, &splits, &pps);
  if (splits == 1) return 0;
  return (size_t)T * n_heads * splits * (MSI_HEAD_DIM + 2) * sizeof(float);
}

extern "C" int msi_decode_attention(const void* q, const void* k_cache, const void* v_cache, int64_t num_pages,
                                    const int32_t* block_table, int max_pages, const int32_t* seq_lens, int T,
                                    int n_heads, int n_kv, float scale, void* out, void* workspace,
                                    size_t ws_bytes, void* stream) {
  MSI_REQUIRE(T >= 0 && n_kv > 0 && n_heads > 0 && n_heads % n_kv == 0 && n_heads / n_kv <= 16,
              "decode_attention: need n_heads = G * n_kv with G <= 16");
  MSI_REQUIRE(max_pages > 0 && num_pages > 0 && num_pages * n_kv * MSI_KV_PAGE < (1LL << 31),
              "decode_attention: bad page counts (rows must fit int32)");
  MSI_REQUIRE(q && k_cache && v_cache && block_table && seq_lens && out, "decode_attention: null pointer");
  MSI_REQUIRE(((uintptr_t)k_cache % 16) == 0 && ((uintptr_t)v_cache % 16) == 0, "decode_attention: caches not 16B aligned");
  if (T == 0) return 0;
  int splits, pps;
  choose_splits(T, n_kv, max_pages, &splits, &pps);
  const size_t need = msi_decode_attention_workspace(T, n_heads, n_kv, max_pages);
  MSI_REQUIRE(ws_bytes >= need && (need == 0 || workspace), "decode_attention: workspace too small (%zu < %zu)",
              ws_bytes, need);
  const uint64_t rows = (uint64_t)num_pages * n_kv * MSI_KV_PAGE;
  // tiny cache of encoded maps (eager calls re-use the same cache tensors)
  static thread_local struct { const void* p; uint64_t rows; uint32_t box; CUtensorMap m; } cache[8];
  static thread_local int next = 0;
  auto lookup = [&](const void* p, uint32_t box, CUtensorMap* m) -> int {
    for (auto& c : cache)
      if (c.p == p && c.rows == rows && c.box == box) {
        *m = c.m;
        return 0;
      }
    int rc = kv_tmap(m, p, rows, box);
    if (rc) return rc;
    cache[next] = {p, rows, box, *m};
    next = (next + 1) % 8;
    return 0;
  };
  CUtensorMap tk, tv, tk16, tv16;  // full-page boxes and 16-row boxes (partial last pages)
  int rc = lookup(k_cache, MSI_KV_PAGE, &tk);
  if (!rc) rc = lookup(v_cache, MSI_KV_PAGE, &tv);
  if (!rc) rc = lookup(k_cache, 16, &tk16);
  if (!rc) rc = lookup(v_cache, 16, &tv16);
  if (rc) return rc;
  if (int arc = smem_attr(reinterpret_cast<const void*>(decode_attn_kernel), kSmem)) return arc;
  AttnArgs a;
  a.q = (const __nv_bfloat16*)q;
  a.bt = block_table;
  a.lens = seq_lens;
  a.out = (__nv_bfloat16*)out;
  a.part_o = (float*)workspace;
  a.part_ml = splits > 1 ? a.part_o + (size_t)T * n_heads * splits * MSI_HEAD_DIM : nullptr;
  a.max_pages = max_pages;
  a.T = T;
  a.n_heads = n_heads;
  a.n_kv = n_kv;
  a.G = n_heads / n_kv;
  a.splits = splits;
  a.pps = pps;
  a.scale_log2 = scale * 1.4426950408889634f;
  const long grid = (long)T * n_kv * splits;
  MSI_REQUIRE(grid < (1L << 31), "decode_attention: grid too large");
  cudaStream_t st = (cudaStream_t)stream;
  MSI_CUDA(launch_k(decode_attn_kernel, dim3((unsigned)grid), dim3(kThreads), kSmem, st, tk, tv, tk16, tv16, a));
  rc = check_launch("decode_attn_kernel");
  if (rc || splits == 1) return rc;
  MSI_CUDA(launch_k(attn_split_combine_kernel, dim3((unsigned)((size_t)T * n_heads)), dim3(MSI_HEAD_DIM), 0, st,
                    (const float*)a.part_o, (const float*)a.part_ml, splits, a.out));
  return check_launch("attn_split_combine_kernel");
}
