// expert_gemm.cu -- expert FFN as two grouped GEMMs on tcgen05 / TMEM / TMA,
// and the attention stage's dense projections on the same kernel.
//
// PAPER.md:285-286 (FFN Input (b_e,h)x(h,h'), FFN Output (b_e,h')x(h',h)),
// SwiGLU per BASELINE north_star.  Rows of local expert e are one compact
// segment starting at a 128-row aligned seg_start[e] (several senders'
// receive regions are gathered there first, gather_regions_kernel), so every
// 128-row M tile belongs to exactly one expert.
//
//   GEMM1  A = X [rows][H], B = W13[e] [2H'][H] (gate/up interleaved in
//          64-row blocks, msi_pack_w13)  ->  epilogue H = bf16(silu(G) * U)
//   GEMM2  A = hbuf [rows][H'], B = W2[e] [H][H']  ->  epilogue stores every
//          Y row over its own X in the receive region (local HBM); the last
//          CTA releases the attention GPUs' arrival counters, whose combine
//          pulls the rows over NVLink (N2M leg).
//   dense  (E_l = 1) the attention projections: QKV with RoPE + paged-KV
//          append in the epilogue (mode 2), O projection + residual (mode 1),
//          attention-TP all-gather (per-shard A maps over NVLink) and
//          reduce-scatter (mode 3, peer stores).
//
// Kernel shape: persistent, one CTA (CG=1) or CTA pair (CG=2, the default:
// tcgen05.mma.cta_group::2, 256x256 tiles, half pairs for odd 128-row
// tails) per SM (pair), 256 threads, warp-specialized:
//   warp 0  TMA producer: A 128x64 + B (256/CG)x64 bf16 per stage, 128B
//           swizzle, 6-stage (CG=2) / 4-stage (CG=1) mbarrier ring
//   warp 1  MMA issuer (one thread of the leader CTA): kind::f16 M=128/256
//           N=256 K=16, fp32 accumulators in TMEM, 2 accumulator buffers
//           (512 TMEM columns) so the epilogue of tile i overlaps the MMAs of
//           tile i+1
//   warp 2  TMEM allocator
//   warps 4-7 epilogue: tcgen05.ld 32x32b -> registers -> swizzled smem
//           staging -> coalesced 256 B row stores (local or NVLink peer)
// Tiles are taken in order (expert-major, then N tile, then M tile) from a
// dynamic scheduler, so CTAs that run together share one expert's B tiles
// in L2.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "gemm.h"

namespace msi {
namespace {

#ifndef MSI_GEMM_PROF  // 1 = MMA-issuer wait profile (diagnostic builds only)
#define MSI_GEMM_PROF 0
#endif
#if MSI_GEMM_PROF
// [0] cycles waiting for operand stages, [1] waiting for a free accumulator,
// [2] MMA-issuer loop cycles, [3] tiles, summed over leaders
__device__ unsigned long long g_gemm_prof[4];
#endif
#ifndef MSI_GEMM_PARAM_QUAL
#define MSI_GEMM_PARAM_QUAL __grid_constant__  // (A/B builds: -DMSI_GEMM_PARAM_QUAL=)
#endif

constexpr int BM = 128, BN = 256, BK = 64;
constexpr int EPI_WARP_BYTES = 32 * 256;  // 32 rows x 128 bf16
#ifndef MSI_EPI_DIRECT  // 1 = CTA-pair epilogue stores rows from registers (no smem staging: one more operand stage)
#define MSI_EPI_DIRECT 0
#endif
constexpr int kThreads = 256;
constexpr int TMEM_COLS = 512;
constexpr int TRING = 4;  // tile ids in flight between the scheduler and the roles

// Per-CTA-group configuration.  CG=1: one CTA computes a 128x256 tile from
// A 128x64 + B 256x64 per stage (48 KB).  CG=2: a CTA pair computes a 256x256
// tile with tcgen05.mma.cta_group::2; each CTA stages its 128 A rows and half
// of B (128 rows) -- 32 KB -- so per-SM shared-memory traffic per MAC is 2/3
// of the CG=1 kernel's and 6 stages fit.
// MAXE = capacity of the per-expert segment table in shared memory; the
// 256-expert variant (fine-grained MoE on few GPUs) gives one pipeline stage
// to the larger table.
template <int CG, int MAXE>
struct Cfg {
  static constexpr bool DIRECT = MSI_EPI_DIRECT && CG == 2;
  static constexpr int STAGES = (CG == 1 ? 4 : 6) - (MAXE > MSI_SMALL_LOCAL_EXPERTS ? 1 : 0) + (DIRECT ? 1 : 0);
  static constexpr int EPI_BYTES = DIRECT ? 0 : 4 * EPI_WARP_BYTES;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_ROWS = BN / CG;
  static constexpr int B_BYTES = B_ROWS * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr size_t SMEM = 1024 /*align*/ + (size_t)STAGES * STAGE_BYTES + EPI_BYTES + 256;
};

template <int MAXE>
struct SegInfo {
  int total[MAXE];
  int start[MAXE];
  int tile0[MAXE + 1];  // first tile of expert e
  int mtiles[MAXE];     // M tiles (CG=1) or M-tile pairs (CG=2)
};

// Receive regions: first virtual row of each sender in local expert e (the
// exclusive prefix of its per-sender counts, read from the count table -- a
// few L2 hits per tile; shared memory has no room left for a table).
__device__ __forceinline__ void load_pre(const GemmParams& p, int e, int (&pre)[MSI_MAX_RANKS + 1]) {
  uint32_t c[MSI_MAX_RANKS];
#pragma unroll
  for (int s = 0; s < MSI_MAX_RANKS; ++s)
    c[s] = s < p.n_src ? (uint32_t)ld_relaxed_sys64(p.cntab + (size_t)s * p.E + p.e0 + e) : 0u;
  pre[0] = 0;
#pragma unroll
  for (int s = 0; s < MSI_MAX_RANKS; ++s) pre[s + 1] = pre[s] + (int)c[s];
}

// A-operand boxes of 128, 64, ..., 1 rows (SW128, 64 columns): a tile's rows
// are loaded as runs of the (expert, sender) receive regions, each run split
// into power-of-two boxes.  The 128-B swizzle is applied by shared-memory
// address (scripts/probe_tma_runs.cu), so a box may land at any row offset.
struct AMaps {
  CUtensorMap m[8];  // m[i]: box of 128 >> i rows
};
constexpr int kMaxPieces = 48;

__device__ __forceinline__ const CUtensorMap* a_box_map(const AMaps& am, uint32_t z) {
  switch (z) {  // constant indices (once per tile)
    case 0: return &am.m[0]; case 1: return &am.m[1]; case 2: return &am.m[2]; case 3: return &am.m[3];
    case 4: return &am.m[4]; case 5: return &am.m[5]; case 6: return &am.m[6]; default: return &am.m[7];
  }
}

// TMA load of A box `z` (128 >> z rows), for tiles made of several runs.
// The producer is one thread whose per-k-block issue cost bounds the MMA
// rate, so single-run tiles (the common case) resolve their box once per
// tile and take the same two-load path as compact rows.
template <bool PAIR>
__device__ __forceinline__ void tma_a_box(const AMaps& am, uint32_t z, void* dst, int c0, int c1, uint64_t* bar) {
#define MSI_TMA_A(I)                                                  \
  case I:                                                             \
    if constexpr (PAIR) tma_load_2d_pair(dst, &am.m[I], c0, c1, bar); \
    else tma_load_2d(dst, &am.m[I], c0, c1, bar);                     \
    break;
  switch (z) { MSI_TMA_A(0) MSI_TMA_A(1) MSI_TMA_A(2) MSI_TMA_A(3) MSI_TMA_A(4) MSI_TMA_A(5) MSI_TMA_A(6) MSI_TMA_A(7) }
#undef MSI_TMA_A
}  // >= the most power-of-two runs 8 senders can cut 128 rows into

// Row runs of this CTA's share [v0, v0 + nrows) of expert e's virtual rows,
// as power-of-two boxes written to shared memory: piece = (smem row | box
// index << 8, global row).  Runs before the last are cut exactly; the last
// run takes one box rounded up to a power of two when it fits the tile (the
// rows past the run are never stored by the epilogue -- the same over-read
// as compact rows' tail tiles), so a tile of one run is one box.  Returns
// the bytes the boxes load (pieces == nullptr: only that, for the peer CTA).
// 8 senders cut 128 rows into at most ~36 boxes.
template <int MAXE>
__device__ __forceinline__ uint32_t plan_pieces(const SegInfo<MAXE>& sg, const GemmParams& p, int e,
                                                const int (&pre)[MSI_MAX_RANKS + 1], int v0, int nrows, uint2* pieces,
                                                int& npieces) {
  npieces = 0;
  uint32_t rows = 0;
  const int end = min(v0 + nrows, sg.total[e]);
#pragma unroll
  for (int s = 0; s < MSI_MAX_RANKS; ++s) {
    if (s >= p.n_src) break;
    const int a = max(v0, pre[s]), b = min(end, pre[s + 1]);
    if (a >= b) continue;
    int off = a - v0, len = b - a;
    long long row = ((long long)e * p.n_src + s) * p.cap_s + (a - pre[s]);
    if (b == end) {  // the tile's last run: one box if the rounded-up size fits
      const int up = len <= 1 ? 1 : 1 << (32 - __clz(len - 1));
      if (off + up <= nrows && up <= 128) len = up;
    }
    while (len > 0 && npieces < kMaxPieces) {
      const int lg = 31 - __clz(min(len, 128));  // largest power of two <= len
      if (pieces) pieces[npieces] = make_uint2((uint32_t)off | ((uint32_t)(7 - lg) << 8), (uint32_t)row);
      ++npieces;
      off += 1 << lg;
      row += 1 << lg;
      len -= 1 << lg;
      rows += 1u << lg;
    }
  }
  return rows * (BK * 2);
}

template <int MAXE>
__device__ __forceinline__ void decode_tile(const SegInfo<MAXE>& s, int E_l, int tau, int& e, int& n, int& m) {
  int lo = 0, hi = E_l - 1;  // last e with tile0[e] <= tau (binary search, E_l up to 256)
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (s.tile0[mid] <= tau) lo = mid;
    else hi = mid - 1;
  }
  e = lo;
  const int local = tau - s.tile0[e];
  n = local / s.mtiles[e];
  m = local - n * s.mtiles[e];
}

// CTA-pair kernels only: the last unit of a segment with an odd number of
// 128-row tiles is a "half pair" -- an M = 128 pair MMA (64 rows per CTA),
// which costs half of an M = 256 one, so odd tiles are not padded to 256.
// Its accumulator is folded in TMEM: row r of the CTA's 64 rows holds N
// columns [0,128) in lane r and [128,256) in lane 64 + r (measured,
// scripts/probe_tmem_pair_m128.cu).
template <int MAXE>
__device__ __forceinline__ bool half_pair_rows(const SegInfo<MAXE>& s, int e, int m) {
  const int mt = (s.total[e] + BM - 1) / BM;
  return (mt & 1) && m == s.mtiles[e] - 1;
}

// QD (quad, CG = 2 only): a cluster of two CTA pairs on N tiles 2j and 2j+1
// of the same (expert, M unit).  Their A slabs are identical, so each CTA
// loads half of its slab and multicasts it to the same-rank CTA of the other
// pair: A traffic from L2 halves (the kernel is L2-bandwidth-bound at
// 256 x 256 pair tiles).  Operand stages are released to all four CTAs.
template <int CG, int MAXE, bool QD = false>
__global__ void __launch_bounds__(kThreads, 1)
grouped_gemm_kernel(const __grid_constant__ AMaps am, const __grid_constant__ CUtensorMap tmB,
                    const MSI_GEMM_PARAM_QUAL GemmParams p) {
  const CUtensorMap& tmA = am.m[0];
  const CUtensorMap& tmA64 = am.m[1];
  using C = Cfg<CG, MAXE>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                                  // STAGES x (A | B) per stage
  uint8_t* sEpi = smem + STAGES * C::STAGE_BYTES;      // 4 x 8 KB epilogue staging
  uint64_t* bars = reinterpret_cast<uint64_t*>(sEpi + C::EPI_BYTES);
  uint64_t* full = bars;                     // [STAGES] (CG=2: the leader's is used)
  uint64_t* empty = bars + STAGES;           // [STAGES]
  uint64_t* tfull = bars + 2 * STAGES;       // [2]
  uint64_t* tempty = bars + 2 * STAGES + 2;  // [2]   (CG=2: the leader's is used)
  uint64_t* qfull = bars + 2 * STAGES + 4;   // [TRING] tile-id ring (per CTA)
  uint64_t* qempty = qfull + TRING;          // [TRING] (CG=2: the leader's is used)
  __shared__ int s_tau[TRING];
  __shared__ uint32_t s_tmem;
  __shared__ SegInfo<MAXE> seg;
  __shared__ int s_last, s_abort;
  __shared__ uint2 s_pieces[kMaxPieces];  // producer: A runs of the current tile

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = CG == 2 ? cluster_ctarank() : 0;  // CTA within the cluster
  const uint32_t rank = crank & 1;                          // CTA within the pair
  const int pr = QD ? (int)(crank >> 1) : 0;                // pair within the quad
  const bool leader = rank == 0;
  const int nunits = QD ? (int)(gridDim.x >> 2) : CG == 2 ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  pdl_trigger();  // the next kernel (GEMM2 / combine) may launch and queue now
  pdl_wait();     // everything earlier on the stream is complete and visible
  uint32_t epoch = p.epoch;
  if (p.epoch_src) epoch = resolve_epoch(p.epoch, p.epoch_src, 1u, p.status);

  // ---- wait for the senders' rows (GEMM1 on an expert GPU); in a pair the
  //      leader waits and both CTAs follow its decision ----------------------
  if (threadIdx.x == 0) {
    bool ok = true;
    if (crank == 0) {
      if (blockIdx.x == 0 && p.trace && p.wait_ctr) p.trace[p.trace_slot] = globaltimer();
      ok = !(p.epoch_src && epoch == 0);  // epoch mismatch: abort below
      if (ok && p.wait_ctr) ok = wait_geq(p.wait_ctr, epoch * p.wait_mul, p.timeout_ns, p.status);
      if (!ok) p.status[1] = 1;
      if (ok && p.status && p.status[1]) ok = false;  // an earlier call failed
    }
    s_abort = ok ? 0 : 1;
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    if (CG == 2 || p.a_runs || p.a_shards > 1) tma_prefetch(&am.m[1]);
    if (p.a_runs || p.a_shards > 2) {
      tma_prefetch(&am.m[2]); tma_prefetch(&am.m[3]); tma_prefetch(&am.m[4]);
      tma_prefetch(&am.m[5]); tma_prefetch(&am.m[6]); tma_prefetch(&am.m[7]);
    }
    for (int i = 0; i < STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], QD ? 2 : 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 4 * CG); }
    // ring consumers: MMA thread + 4 epilogue warps (+ the peer's producer
    // and 4 epilogue warps, which arrive on the leader's barrier)
    // (quad: 2 MMA threads, 3 producers, 16 epilogue warps on the quad leader's)
    for (int i = 0; i < TRING; ++i) { mbar_init(&qfull[i], 1); mbar_init(&qempty[i], QD ? 21 : CG == 2 ? 10 : 5); }
    fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (CG == 2) tmem_alloc2<TMEM_COLS>(&s_tmem);
    else tmem_alloc<TMEM_COLS>(&s_tmem);
  }
  tc_fence_before();
  if constexpr (CG == 2) {
    cluster_sync();  // barriers of both CTAs initialised, leader's wait done
    if (crank != 0) {
      if (threadIdx.x == 0) s_abort = (int)ld_shared_cluster_u32(mapa_shared(smem_u32(&s_abort), 0));
      __syncthreads();
    }
  } else {
    __syncthreads();
  }
  tc_fence_after();
  if (threadIdx.x == 0) fence_proxy_async_global();  // rows written by peers are read by TMA
  const uint32_t tmem_base = s_tmem;
  if (s_abort) {  // a wait timed out / epoch mismatch: skip the work, keep the GPU usable
    if constexpr (CG == 2) cluster_sync();
    else __syncthreads();
    if (warp == 2) {
      if constexpr (CG == 2) tmem_dealloc2<TMEM_COLS>(tmem_base);
      else tmem_dealloc<TMEM_COLS>(tmem_base);
    }
    return;
  }

  // ---- segment table (all threads compute the same) -----------------------
  if (blockIdx.x == 0 && threadIdx.x == 0 && p.trace) p.trace[p.trace_slot + 1] = globaltimer();
  // totals: every (sender, expert) count loaded in parallel (no serial chain
  // of system-scope loads), summed in shared memory
  for (int e = threadIdx.x; e < p.E_l; e += blockDim.x) seg.total[e] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < (p.a_shards ? p.E_l : p.dense_rows ? 1 : p.totals ? p.E_l : p.n_a * p.E_l);
       i += blockDim.x) {
    if (p.a_shards) {
      seg.total[i] = p.shard_rows;
    } else if (p.dense_rows) {
      seg.total[0] = (int)p.dense_rows;
    } else if (p.totals) {
      seg.total[i] = p.totals[i];
    } else {
      const int s = i / p.E_l, e = i - s * p.E_l;
      atomicAdd(&seg.total[e], (int)(uint32_t)ld_relaxed_sys64(p.cntab + (size_t)s * p.E + p.e0 + e));
    }
  }
  // every total complete before thread 0 builds the table: with more than 32
  // (expert, sender) entries the adds come from several warps, and a CTA
  // (or the two CTAs of a pair) seeing a partial sum would disagree on the
  // tile list -- the pair then waits on each other forever (found at
  // DeepSeek-V3 shape, 64 local experts x 4 senders)
  __syncthreads();
  if (threadIdx.x == 0) {
    int run_start = 0, run_tile = 0;
    for (int e = 0; e < p.E_l; ++e) {
      const int tot = seg.total[e];
      const int mt = (tot + BM - 1) / BM;
      const int units = (mt + CG - 1) / CG;  // M tiles per CTA or per pair
      seg.start[e] = run_start;
      seg.mtiles[e] = units;
      seg.tile0[e] = run_tile;
      run_start += mt * BM;
      run_tile += units * p.nt;
    }
    seg.tile0[p.E_l] = run_tile;
    if (p.stats && blockIdx.x == 0) {
      unsigned long long rows = 0;
      for (int e = 0; e < p.E_l; ++e) rows += seg.total[e];
      atomicAdd(p.stats, rows);
      atomicAdd(p.stats + 1, 1ull);
    }
  }
  __syncthreads();
  // split-K (mode 4 only): unit tau covers tile tau % ntiles1 over the K
  // range of split tau / ntiles1, written to its own fp32 plane
  const int ksplit = p.ksplit > 1 ? p.ksplit : 1;
  const int ntiles1 = seg.tile0[p.E_l];
  const int ntiles = ntiles1 * ksplit;
  const int kblocks = p.kdim / BK / ksplit;
  auto half_pair = [&](const SegInfo<MAXE>& sg, int e, int m) -> bool {
    if constexpr (CG == 2) return half_pair_rows(sg, e, m);
    else return false;
  };
  // ---- dynamic tile scheduler ------------------------------------------
  // The leader's producer thread takes tile ids in order from p.tile_ctr and
  // publishes them through a TRING-deep ring to every role of the CTA (and of
  // the peer CTA).  Taking tiles in order keeps the CTAs that run together on
  // neighbouring tiles (the M tiles of one N tile share its weights in L2)
  // even though half-pair tiles cost half: a static round-robin drifts
  // apart and re-reads weights from DRAM (measured 2.2x).
  auto publish_tile = [&](int it) -> int {  // leader producer thread only
    const int slot = it % TRING;
    if (it >= TRING) mbar_wait_cluster(&qempty[slot], ((it / TRING) - 1) & 1);
    const uint32_t t = atomicAdd(p.tile_ctr, 1u);
    if (t == (uint32_t)((QD ? ntiles / 2 : ntiles) + nunits - 1)) *p.tile_ctr = 0;  // the launch's last fetch
    s_tau[slot] = (int)t;
    if constexpr (CG == 2) {
      for (uint32_t r = 1; r < (QD ? 4u : 2u); ++r) {
        st_shared_cluster_u32(mapa_shared(smem_u32(&s_tau[slot]), r), t);
        mbar_arrive_cluster(mapa_shared(smem_u32(&qfull[slot]), r));
      }
    }
    mbar_arrive(&qfull[slot]);
    return (int)t;
  };
  auto take_tile = [&](int it, bool arrive) -> int {  // consumers (one call per warp-role and tile)
    const int slot = it % TRING;
    mbar_wait_cluster(&qfull[slot], (it / TRING) & 1);
    const int t = s_tau[slot];
    if (arrive) {
      if constexpr (CG == 2) {
        if (crank == 0) mbar_arrive(&qempty[slot]);
        else mbar_arrive_cluster(mapa_shared(smem_u32(&qempty[slot]), 0));
      } else {
        mbar_arrive(&qempty[slot]);
      }
    }
    return t;
  };
  // quad: the ring carries quad-tile ids (expert, N-tile pair, M unit); this
  // pair's tile is N tile 2j + pr (ntiles = the end sentinel)
  auto pair_tile = [&](int t) -> int {
    if constexpr (!QD) {
      return t;
    } else {
      if (t >= ntiles / 2) return ntiles;
      int lo = 0, hi = p.E_l - 1;  // last e with tile0[e] / 2 <= t
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if ((seg.tile0[mid] >> 1) <= t) lo = mid;
        else hi = mid - 1;
      }
      const int local = t - (seg.tile0[lo] >> 1);
      const int nq = local / seg.mtiles[lo];
      return seg.tile0[lo] + (2 * nq + pr) * seg.mtiles[lo] + (local - nq * seg.mtiles[lo]);
    }
  };

  if (warp == 0) {
    // ===================== TMA producer (both CTAs of a pair) ==============
    // Lane 0 takes tiles, plans them and issues the loads of single-run
    // tiles; a tile of several receive-region runs has its boxes issued by
    // lanes 0..n-1 at once (the single issuing thread bounds the MMA rate).
    int stage = 0;
    uint32_t phase = 0;
    uint2* pieces = s_pieces;
    const uint64_t pol_a = l2_policy_evict_last(), pol_b = l2_policy_evict_first();
    int pre[MSI_MAX_RANKS + 1];
    int pre_e = -1;  // expert whose sender prefix is in pre (tiles arrive expert-major)
    for (int it = 0;; ++it) {
      int tau = 0;
      if (lane == 0) tau = pair_tile(crank == 0 ? publish_tile(it) : take_tile(it, true));
      tau = __shfl_sync(0xffffffffu, tau, 0);
      if (tau >= ntiles) break;
      const int kb0 = (tau / ntiles1) * kblocks;  // split-K: first k-block of this unit
      int e, n, m;
      decode_tile(seg, p.E_l, tau % ntiles1, e, n, m);
      // this CTA's A rows: 128 (full tile / pair) or 64 (half pair: the odd
      // last 128-row tile of a segment split 64/64 over the pair, moved with
      // a 64-row box so the half-cost MMA is not fed a full tile's bytes)
      const bool hp = half_pair(seg, e, m);
      int rowA = (p.a_shards ? 0 : seg.start[e]) + m * CG * BM + (int)rank * (hp ? BM / 2 : BM);
      const int rowB = (p.a_shards ? 0 : e * p.n_total) + n * BN + (int)rank * C::B_ROWS;
      const CUtensorMap* mA = p.a_shards ? a_box_map(am, (uint32_t)e)                 // shard e's own map
                              : (CG == 2 && hp && p.a64) ? &tmA64 : &tmA;               // compact rows
      uint32_t a_bytes = (CG == 2 && hp && p.a64 && !p.a_shards) ? C::A_BYTES / 2 : C::A_BYTES;
      uint32_t a_bytes_pair = 2 * a_bytes;  // both CTAs' A bytes (the leader's barrier counts them)
      int npieces = 0;
      if (p.a_runs && lane == 0) {  // receive regions: only the rows present, as runs
        const int nrows = hp ? BM / 2 : BM;
        const int v0 = m * CG * BM + (int)rank * nrows;
        if (e != pre_e) {
          load_pre(p, e, pre);
          pre_e = e;
        }
        a_bytes = plan_pieces(seg, p, e, pre, v0, nrows, pieces, npieces);
        if constexpr (CG == 2) {  // the peer CTA's boxes (same plan, its rows)
          const int v1 = m * CG * BM + (int)(rank ^ 1) * nrows;
          int n1 = 0;
          a_bytes_pair = a_bytes + plan_pieces(seg, p, e, pre, v1, nrows, nullptr, n1);
        }
        if (npieces == 1) {  // one run from the tile's first row: the compact path with its box
          mA = a_box_map(am, pieces[0].x >> 8);
          rowA = (int)pieces[0].y;
        }
      }
      if (p.a_runs) npieces = __shfl_sync(0xffffffffu, npieces, 0);
      const bool multi = npieces > 1;
      __syncwarp();  // the pieces in shared memory are visible to every lane
      for (int kb = 0; kb < kblocks; ++kb) {
        uint8_t* st = sA + stage * C::STAGE_BYTES;
        if (lane == 0) {
          mbar_wait(&empty[stage], phase ^ 1);
          if constexpr (CG == 2) {
            if (leader) mbar_expect_tx(&full[stage], a_bytes_pair + 2 * C::B_BYTES);
            if (p.l2hint) {  // A (re-read by every N tile) evict-last, B (streamed) evict-first
              if (!multi && a_bytes) tma_load_2d_pair_hint(st, mA, (kb0 + kb) * BK, rowA, &full[stage], pol_a);
              tma_load_2d_pair_hint(st + C::A_BYTES, &tmB, (kb0 + kb) * BK, rowB, &full[stage], pol_b);
            } else {
              if (QD && !hp) {  // half of the slab, to this CTA and its twin in the other pair
                tma_load_2d_pair_mc(st + pr * (C::A_BYTES / 2), &tmA64, (kb0 + kb) * BK, rowA + pr * (BM / 2),
                                    &full[stage], (uint16_t)((1u << rank) | (4u << rank)));
              } else if (!multi && a_bytes) {
                tma_load_2d_pair(st, mA, (kb0 + kb) * BK, rowA, &full[stage]);
              }
              tma_load_2d_pair(st + C::A_BYTES, &tmB, (kb0 + kb) * BK, rowB, &full[stage]);
            }
          } else {
            mbar_expect_tx(&full[stage], a_bytes + C::B_BYTES);
            if (p.l2hint) {
              if (!multi && a_bytes) tma_load_2d_hint(st, mA, (kb0 + kb) * BK, rowA, &full[stage], pol_a);
              tma_load_2d_hint(st + C::A_BYTES, &tmB, (kb0 + kb) * BK, rowB, &full[stage], pol_b);
            } else {
              if (!multi && a_bytes) tma_load_2d(st, mA, (kb0 + kb) * BK, rowA, &full[stage]);
              tma_load_2d(st + C::A_BYTES, &tmB, (kb0 + kb) * BK, rowB, &full[stage]);
            }
          }
        }
        // weights stream from HBM once per N tile: pull the tile p.pfb k-blocks
        // ahead into L2 so the stage's load meets an L2 hit
        if (p.pfb && lane == 0 && kb + p.pfb < kblocks) tma_prefetch_l2_2d(&tmB, (kb0 + kb + p.pfb) * BK, rowB);
        if (multi) {
          __syncwarp();  // the stage is free (lane 0 waited for it)
          for (int i = lane; i < npieces; i += 32) {
            const uint2 pc = pieces[i];
            tma_a_box<CG == 2>(am, pc.x >> 8, st + (pc.x & 0xff) * (BK * 2), kb * BK, (int)pc.y, &full[stage]);
          }
        }
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      __syncwarp();  // the pieces may be rewritten for the next tile
    }
  } else if (warp == 1 && lane == 0 && leader) {
    // ===================== MMA issuer (leader only) =====================
    constexpr uint32_t idesc_full = umma_idesc_bf16(BM * CG, BN);
    constexpr uint32_t idesc_half = umma_idesc_bf16(BM, BN);  // CG = 2 only
    int stage = 0;
    uint32_t phase = 0;
#if MSI_GEMM_PROF
    unsigned long long w_full = 0, w_acc = 0, ntile = 0;
    const long long t_begin = clock64();
#endif
    for (int it = 0;; ++it) {
      const int tau = pair_tile(take_tile(it, true));
      if (tau >= ntiles) break;
      int e_, n_, m_;
      decode_tile(seg, p.E_l, tau % ntiles1, e_, n_, m_);
      const uint32_t idesc = half_pair(seg, e_, m_) ? idesc_half : idesc_full;
      const int acc = it & 1;
      const uint32_t aph = (it >> 1) & 1;
#if MSI_GEMM_PROF
      long long t0 = clock64();
#endif
      mbar_wait(&tempty[acc], aph ^ 1);
#if MSI_GEMM_PROF
      w_acc += clock64() - t0;
      ++ntile;
#endif
      tc_fence_after();
      const uint32_t d = tmem_base + acc * BN;
      for (int kb = 0; kb < kblocks; ++kb) {
#if MSI_GEMM_PROF
        t0 = clock64();
#endif
        mbar_wait(&full[stage], phase);
#if MSI_GEMM_PROF
        w_full += clock64() - t0;
#endif
        tc_fence_after();
        uint8_t* st = sA + stage * C::STAGE_BYTES;
        const uint64_t ad = umma_desc_sw128(st);
        const uint64_t bd = umma_desc_sw128(st + C::A_BYTES);
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {  // +32 B along K inside the 128 B swizzle atom
          if constexpr (CG == 2) mma_bf16_pair(d, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
          else mma_bf16(d, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
        }
        if constexpr (QD) mma_commit_pair_mask(&empty[stage], 0xF);  // both pairs fill every stage
        else if constexpr (CG == 2) mma_commit_pair(&empty[stage]);
        else mma_commit(&empty[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if constexpr (QD) mma_commit_pair_mask(&tfull[acc], (uint16_t)(3u << (2 * pr)));
      else if constexpr (CG == 2) mma_commit_pair(&tfull[acc]);
      else mma_commit(&tfull[acc]);
    }
#if MSI_GEMM_PROF
    atomicAdd(&g_gemm_prof[0], w_full);
    atomicAdd(&g_gemm_prof[1], w_acc);
    atomicAdd(&g_gemm_prof[2], (unsigned long long)(clock64() - t_begin));
    atomicAdd(&g_gemm_prof[3], ntile);
#endif
  } else if (warp >= 4) {
    // ===================== epilogue (both CTAs, own TMEM rows) ============
    // Full tile: warp q owns TMEM lanes [32q, 32q+32) = rows 32q.. of the
    // CTA's 128, all 256 N columns.  Half pair: lanes hold rows (q & 1)*32..
    // of the CTA's 64 and N columns [(q >> 1)*128, +128) (folded layout).
    // GEMM1 N tiles pack [gate 64 | up 64 | gate 64 | up 64] (msi_pack_w13), so
    // every 128-column half holds matching gate/up features.
    const int q = warp & 3;  // TMEM lanes [32q, 32q+32)
    uint8_t* stg = sEpi + q * EPI_WARP_BYTES;
    int pre[MSI_MAX_RANKS + 1];
    int pre_e = -1;  // receive regions: sender prefix of expert pre_e
    for (int it = 0;; ++it) {
      int tau = 0;
      if (lane == 0) tau = pair_tile(take_tile(it, false));
      tau = __shfl_sync(0xffffffffu, tau, 0);
      __syncwarp();
      if (lane == 0) {  // one ring arrival per epilogue warp
        const int slot = it % TRING;
        if constexpr (CG == 2) {
          if (crank == 0) mbar_arrive(&qempty[slot]);
          else mbar_arrive_cluster(mapa_shared(smem_u32(&qempty[slot]), 0));
        } else {
          mbar_arrive(&qempty[slot]);
        }
      }
      if (tau >= ntiles) break;
      const int ks = tau / ntiles1;  // split-K plane (mode 4)
      int e, n, m;
      decode_tile(seg, p.E_l, tau % ntiles1, e, n, m);
      const bool hp = half_pair(seg, e, m);
      const int rowbase = hp ? m * CG * BM + (int)rank * (BM / 2) : (m * CG + (int)rank) * BM;
      const int rowsub = hp ? (q & 1) * 32 : q * 32;
      const int nh = hp ? (q >> 1) : 0;  // N half held by this warp (half pair)
      const int acc = it & 1;
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
      const int row_local = rowbase + rowsub + lane;                // row within expert segment
      const int row_global = (p.a_shards ? e * p.shard_rows : seg.start[e]) + row_local;  // row in recv / hbuf
      const int valid_rows = min(32, max(0, seg.total[e] - (rowbase + rowsub)));
      // output columns of this warp: mode 0 writes 128 features per tile
      // (64 per N half), mode 1 writes 256 columns (128 per N half)
      const int colofs = (p.mode == 0) ? nh * 64 : nh * 128;

      char* rowdst = nullptr;
      int pos_t = 0, page_t = 0;  // mode 2: the row's token position and its KV page
      if (row_local < seg.total[e]) {
        if (p.mode == 0) {
          rowdst = reinterpret_cast<char*>(p.out) + ((size_t)row_global * p.out_ld + (size_t)n * (BN / 2) + colofs) * 2;
        } else if (p.mode == 3) {  // attention-TP reduce-scatter: the token's shard owner
          const int sh = row_global / p.shard_rows;
          rowdst = reinterpret_cast<char*>(p.peer_out[sh]) +
                   ((size_t)(row_global - sh * p.shard_rows) * p.out_ld + (size_t)n * BN + colofs) * 2;
        } else if (p.mode == 2) {  // per-head destinations below
          pos_t = p.pos[row_global];
          page_t = p.block_table[(size_t)row_global * p.max_pages + pos_t / MSI_KV_PAGE];
          rowdst = reinterpret_cast<char*>(p.q_out);
        } else if (p.n_src) {  // receive regions: Y of virtual row row_local replaces its X in place
          if (e != pre_e) {
            load_pre(p, e, pre);
            pre_e = e;
          }
          int s = 0, base = 0;
#pragma unroll
          for (int j = 1; j < MSI_MAX_RANKS; ++j)  // last sender whose first row is <= row_local
            if (j < p.n_src && pre[j] <= row_local) { s = j; base = pre[j]; }
          const long long rrow = ((long long)e * p.n_src + s) * p.cap_s + (row_local - base);
          rowdst = reinterpret_cast<char*>(p.out) + ((size_t)rrow * p.out_ld + (size_t)n * BN + colofs) * 2;
        } else {
          rowdst = reinterpret_cast<char*>(p.out) + ((size_t)row_global * p.out_ld + (size_t)n * BN + colofs) * 2;
        }
      }
      // 256-byte row segments (mode 1/2 full: 2, mode 1/2 half / mode 0 full: 1)
      // or one 128-byte segment (mode 0 half)
      const int segs = (p.mode != 0 && !hp) ? 2 : 1;
      const bool narrow = (p.mode == 0 && hp);
      char* segdst_l = nullptr;  // DIRECT: this lane's row segment
      auto stage = [&](int cc, const uint32_t (&pk)[16]) {  // 32 bf16 of the lane's row -> swizzled staging
        if constexpr (C::DIRECT) {  // or straight to the row's destination (64 B per lane)
          if (segdst_l && lane < valid_rows) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              st_v4(segdst_l + (cc * 4 + j) * 16, make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]));
          }
          return;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int u = cc * 4 + j;
          uint4 val = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
          const int sw = narrow ? (u ^ (lane & 7)) : (u ^ (lane & 15));
          *reinterpret_cast<uint4*>(stg + lane * 256 + sw * 16) = val;
        }
      };
      for (int sgi = 0; sgi < segs; ++sgi) {
        // mode 2: the segment's 128 columns are one head of q | k | v
        const int head = p.mode == 2 ? n * 2 + (hp ? nh : sgi) : 0;
        const bool rope = p.mode == 2 && head < p.n_heads + p.n_kv;
        char* segdst = nullptr;
        if (rowdst) {
          if (p.mode == 2) {
            __nv_bfloat16* d;
            if (head < p.n_heads) {
              d = p.q_out + ((size_t)row_global * p.n_heads + head) * 128;
            } else {
              const bool isk = head < p.n_heads + p.n_kv;
              const int kvh = head - p.n_heads - (isk ? 0 : p.n_kv);
              d = (isk ? p.k_cache : p.v_cache) +
                  (((size_t)page_t * p.n_kv + kvh) * MSI_KV_PAGE + pos_t % MSI_KV_PAGE) * 128;
            }
            segdst = reinterpret_cast<char*>(d);
          } else {
            segdst = rowdst + sgi * 256;
          }
        }
        segdst_l = segdst;
        const __nv_bfloat16* rsrc = (p.mode == 1 && p.resid && rowdst)
            ? p.resid + (size_t)row_global * p.resid_ld + (size_t)n * BN + colofs + sgi * 128 : nullptr;
        if (valid_rows > 0) {
          const int nchunk = narrow ? 2 : 4;
#pragma unroll 1
          for (int c = 0; c < nchunk; ++c) {
            uint32_t packed[16];
            if (p.mode == 0) {
              // features 32c.. of this tile (half pair: of this N half):
              // gate at column gc, up at gc + 64
              const int gc = hp ? c * 32 : (c < 2 ? c * 32 : 128 + (c - 2) * 32);
              uint32_t g[32], u[32];
              tmem_ld32(tbase + gc, g);
              tmem_ld32(tbase + gc + 64, u);
              tmem_wait_ld();
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                float g0 = __uint_as_float(g[2 * j]), g1 = __uint_as_float(g[2 * j + 1]);
                float u0 = __uint_as_float(u[2 * j]), u1 = __uint_as_float(u[2 * j + 1]);
                float h0 = g0 / (1.0f + __expf(-g0)) * u0;
                float h1 = g1 / (1.0f + __expf(-g1)) * u1;
                packed[j] = pack_bf16x2(h0, h1);
              }
            } else if (p.mode == 4) {
              // fp32 rows (router logits): the lane's 32 consecutive columns
              // straight from registers, 128 B per lane and chunk
              uint32_t v[32];
              tmem_ld32(tbase + sgi * 128 + c * 32, v);
              tmem_wait_ld();
              if (row_local < seg.total[e]) {
                uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<float*>(p.out) + (size_t)ks * p.plane +
                                                      (size_t)row_global * p.out_ld + (size_t)n * BN + colofs +
                                                      sgi * 128 + c * 32);
#pragma unroll
                for (int j = 0; j < 8; ++j) dst[j] = make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
              }
              continue;
            } else if (rope) {
              // rotate-half RoPE pairs dims (i, i + 64): chunks c and c + 2
              // together; same arithmetic as rope_append_kernel on the
              // bf16-rounded projection (attention.cu)
              if (c >= 2) continue;
              uint32_t lo[32], hi[32], rh[16];
              tmem_ld32(tbase + sgi * 128 + c * 32, lo);
              tmem_ld32(tbase + sgi * 128 + 64 + c * 32, hi);
              tmem_wait_ld();
              const float fp = (float)pos_t;
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                float r0[2], r1[2];
#pragma unroll
                for (int b = 0; b < 2; ++b) {
                  const float inv = p.rope.v[c * 32 + 2 * j + b];  // (grid-constant parameter: no local copy)
                  float sn, cs;
                  sincosf(fp * inv, &sn, &cs);
                  const float x0 = __bfloat162float(__float2bfloat16_rn(__uint_as_float(lo[2 * j + b])));
                  const float x1 = __bfloat162float(__float2bfloat16_rn(__uint_as_float(hi[2 * j + b])));
                  r0[b] = x0 * cs - x1 * sn;
                  r1[b] = x1 * cs + x0 * sn;
                }
                packed[j] = pack_bf16x2(r0[0], r0[1]);
                rh[j] = pack_bf16x2(r1[0], r1[1]);
              }
              stage(c + 2, rh);
            } else {
              uint32_t v[32];
              tmem_ld32(tbase + sgi * 128 + c * 32, v);
              if (p.resid) {  // residual (O projection): out = bf16(acc + x), one rounding
                // (warp-uniform branch: tcgen05.wait::ld is .sync.aligned;
                // lanes past the last row load nothing)
                uint32_t r[16];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const uint4 q4 = rsrc ? ld_nc_v4(rsrc + c * 32 + 8 * j) : make_uint4(0u, 0u, 0u, 0u);
                  r[4 * j] = q4.x; r[4 * j + 1] = q4.y; r[4 * j + 2] = q4.z; r[4 * j + 3] = q4.w;
                }
                tmem_wait_ld();
#pragma unroll
                for (int j = 0; j < 16; ++j)
                  packed[j] = pack_bf16x2(__uint_as_float(v[2 * j]) + bf16lo(r[j]),
                                          __uint_as_float(v[2 * j + 1]) + bf16hi(r[j]));
              } else {
                tmem_wait_ld();
#pragma unroll
                for (int j = 0; j < 16; ++j)
                  packed[j] = pack_bf16x2(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1]));
              }
            }
            stage(c, packed);
          }
        }
        if (sgi == segs - 1) {
          // accumulator fully read: hand the TMEM buffer back to the MMA warp
          // (one arrival per warp; a pair's peer arrives on the leader's barrier)
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (CG == 2) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), crank & ~1u));
            else mbar_arrive(&tempty[acc]);
          }
        }
        __syncwarp();
        if (p.mode == 4 || C::DIRECT) continue;  // rows already stored from registers
        if (!narrow) {
          // ---- coalesced row stores: 2 rows per instruction, 256 B per row ----
          const int u = lane & 15;
          for (int r0 = 0; r0 < valid_rows; r0 += 2) {
            const int r = r0 + (lane >> 4);
            char* dst = reinterpret_cast<char*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(segdst), r & 31));
            if (r < valid_rows) {
              uint4 val = *reinterpret_cast<const uint4*>(stg + r * 256 + ((u ^ (r & 15)) * 16));
              st_v4(dst + u * 16, val);
            }
          }
        } else {
          // ---- 128 B rows: 4 rows per instruction ----
          const int u = lane & 7;
          for (int r0 = 0; r0 < valid_rows; r0 += 4) {
            const int r = r0 + (lane >> 3);
            char* dst = reinterpret_cast<char*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(segdst), r & 31));
            if (r < valid_rows) {
              uint4 val = *reinterpret_cast<const uint4*>(stg + r * 256 + ((u ^ (r & 7)) * 16));
              st_v4(dst + u * 16, val);
            }
          }
        }
        __syncwarp();
      }
    }
  }

  // ---- teardown + completion signal --------------------------------------
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync();  // the leader's last commits target both CTAs
  else __syncthreads();
  if (warp == 2) {
    if constexpr (CG == 2) tmem_dealloc2<TMEM_COLS>(tmem_base);
    else tmem_dealloc<TMEM_COLS>(tmem_base);
  }
  if (p.n_sig > 0 && threadIdx.x == 0) {
    __threadfence_system();
    s_last = (atomicAdd(p.ticket, 1u) == gridDim.x - 1);
    if (s_last) {
      *p.ticket = 0;
      if (p.epoch_store) *p.epoch_store = epoch;
      if (p.trace) p.trace[p.trace_slot + 2] = globaltimer();
      fence_sys();
      for (int i = 0; i < p.n_sig; ++i) red_release_sys_add(p.sig[i], 1u);
    }
  }
}

// ------------------------------------------------ region gather ----------
// Several senders' receive regions per expert -> one compact 128-row aligned
// segment per expert, so GEMM1 loads every A tile with one 128-row box.
// (Loading a tile that straddles two regions as runs of power-of-two boxes
// costs ~8 TMA issues per k-block; measured 1.25-2x slower GEMM1 at 2-8
// senders, scripts/ab_ffn_regions_1gpu.py.)  HBM-bound copy of the rows
// (2 * rows * H * 2 bytes), one warp per row; optionally waits for the
// senders' arrivals first (the expert_wait of msi_expert_ffn).
constexpr int kGatherThreads = 512;

__global__ void __launch_bounds__(kGatherThreads)
gather_regions_kernel(const __nv_bfloat16* __restrict__ recv, const uint64_t* cntab, int E, int e0, int n_src,
                      int E_l, long long cap_s, int H, __nv_bfloat16* __restrict__ xc, const uint32_t* wait_ctr,
                      uint32_t epoch, const uint32_t* epoch_src, uint32_t wait_mul, uint64_t timeout_ns,
                      int32_t* status) {
  extern __shared__ int g_sm[];
  int* vpre = g_sm;                    // [E_l + 1] exclusive prefix of expert totals (virtual rows)
  int* cstart = vpre + E_l + 1;        // [E_l] compact 128-aligned segment start
  int* spre = cstart + E_l;            // [E_l][n_src + 1] sender prefix within the expert
  __shared__ int s_abort;
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x == 0) {
    bool ok = true;
    if (wait_ctr) {
      if (epoch_src) epoch = resolve_epoch(epoch, epoch_src, 1u, status);
      ok = epoch != 0 && wait_geq(wait_ctr, epoch * wait_mul, timeout_ns, status);
      if (!ok) status[1] = 1;
    }
    s_abort = ok ? 0 : 1;
  }
  __syncthreads();
  if (s_abort) return;
  for (int e = threadIdx.x; e < E_l; e += blockDim.x) {
    int* sp = spre + e * (n_src + 1);
    int run = 0;
    sp[0] = 0;
    for (int s = 0; s < n_src; ++s) {
      run += (int)(uint32_t)ld_relaxed_sys64(cntab + (size_t)s * E + e0 + e);
      sp[s + 1] = run;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // E_l <= 256: serial scan
    int v = 0, c = 0;
    for (int e = 0; e < E_l; ++e) {
      const int t = spre[e * (n_src + 1) + n_src];
      vpre[e] = v;
      cstart[e] = c;
      v += t;
      c += (t + 127) / 128 * 128;
    }
    vpre[E_l] = v;
  }
  __syncthreads();
  const int total = vpre[E_l];
  const int lane = threadIdx.x & 31;
  const int nvec = H / 8;  // 16-byte vectors per row
  for (int v = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); v < total;
       v += gridDim.x * (blockDim.x >> 5)) {
    int lo = 0, hi = E_l - 1;  // last expert with vpre[e] <= v
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (vpre[mid] <= v) lo = mid;
      else hi = mid - 1;
    }
    const int e = lo, ve = v - vpre[e];
    const int* sp = spre + e * (n_src + 1);
    int s = 0;
    while (s + 1 < n_src && sp[s + 1] <= ve) ++s;
    const uint4* src = reinterpret_cast<const uint4*>(recv + ((size_t)(e * n_src + s) * cap_s + (ve - sp[s])) * H);
    uint4* dst = reinterpret_cast<uint4*>(xc + ((size_t)cstart[e] + ve) * H);
    int i = lane;
    for (; i + 96 < nvec; i += 128) {  // 4 loads in flight per lane
      const uint4 a = src[i], b = src[i + 32], c = src[i + 64], d = src[i + 96];
      dst[i] = a; dst[i + 32] = b; dst[i + 64] = c; dst[i + 96] = d;
    }
    for (; i < nvec; i += 32) dst[i] = src[i];
  }
}

// ---------------------------------------------------------- tensor maps ----
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}

int make_tmap(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint32_t box_inner,
              uint32_t box_outer) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return MSI_EDRIVER;
  }
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d): inner=%llu outer=%llu", (int)r,
              (unsigned long long)inner, (unsigned long long)outer);
    return MSI_EDRIVER;
  }
  return 0;
}

__global__ void pack_w13_kernel(const uint4* __restrict__ gate, const uint4* __restrict__ up,
                                uint4* __restrict__ out, int E_l, int inter, int hidden) {
  // out[e][256 j + 64 b + i] = (b even ? gate : up)[e][128 j + 64 (b >> 1) + i]
  // i.e. every 256-row N tile is [gate 64 | up 64 | gate 64 | up 64] of 128 features
  const size_t row_vec = (size_t)hidden / 8;
  const size_t total = (size_t)E_l * 2 * inter * row_vec;
  for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < total; v += (size_t)gridDim.x * blockDim.x) {
    const size_t row = v / row_vec, col = v % row_vec;
    const size_t e = row / (2 * inter), r = row % (2 * inter);
    const size_t blk = r / 256, i = r % 256, b = i / 64;
    const uint4* src = (b & 1) ? up : gate;
    const size_t srow = e * inter + blk * 128 + (b >> 1) * 64 + (i & 63);
    out[v] = src[srow * row_vec + col];
  }
}

}  // namespace

// Half-pair tiles load their 64 A rows per CTA with a 64-row TMA box
// (MSI_GEMM_A64=1; 0 = the 128-row box, for A/B runs).
bool half_pair_box64() {
  const char* e = getenv("MSI_GEMM_A64");  // read per launch: bench_gemm.py --ab-env flips it
  return e && e[0] == '1';
}

// MSI_GEMM_L2HINT=1: TMA loads carry L2 eviction priorities (A evict-last,
// B evict-first); read per launch for A/B runs
bool l2_hints() {
  const char* e = getenv("MSI_GEMM_L2HINT");
  return e && e[0] == '1';
}

int num_sms() {
  static int n[64] = {};  // per device (all B200s have 148; no race: idempotent)
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!n[dev]) cudaDeviceGetAttribute(&n[dev], cudaDevAttrMultiProcessorCount, dev);
  return n[dev];
}

int gather_regions(const void* recv, const uint64_t* cntab, int E, int e0, int n_src, int E_l, long long cap_s,
                   int H, void* xc, const uint32_t* wait_ctr, uint32_t epoch, const uint32_t* epoch_src,
                   uint32_t wait_mul, uint64_t timeout_ns, int32_t* status, cudaStream_t st) {
  MSI_REQUIRE(E_l >= 1 && E_l <= MSI_MAX_LOCAL_EXPERTS && n_src >= 1 && n_src <= MSI_MAX_RANKS && H % 8 == 0,
              "gather_regions: bad shape");
  const size_t smem = (size_t)(E_l + 1 + E_l + E_l * (n_src + 1)) * sizeof(int);
  if (int arc = smem_attr(reinterpret_cast<const void*>(gather_regions_kernel), smem)) return arc;
  MSI_CUDA(launch_k(gather_regions_kernel, dim3(2 * num_sms()), dim3(kGatherThreads), smem, st,
                    reinterpret_cast<const __nv_bfloat16*>(recv), cntab, E, e0, n_src, E_l, cap_s, H,
                    reinterpret_cast<__nv_bfloat16*>(xc), wait_ctr, epoch, epoch_src, wait_mul, timeout_ns, status));
  return check_launch("gather_regions_kernel");
}

template <int CG, int MAXE, bool QD = false>
int launch_cg(const GemmLaunch& L, cudaStream_t st) {
  using C = Cfg<CG, MAXE>;
  AMaps am;
  CUtensorMap tb;
  int rc = 0;
  if (L.p.a_shards) {  // one 128-row-box map per shard (node peer)
    MSI_REQUIRE(L.p.a_shards == L.p.E_l && L.p.a_shards <= 8 && !L.p.a_runs, "grouped_gemm: bad shard setup");
    for (int i = 0; i < 8 && !rc; ++i)
      rc = make_tmap(&am.m[i], L.a_shard[i < L.p.a_shards ? i : 0], (uint64_t)L.p.kdim, (uint64_t)L.a_rows, BK, BM);
  } else {
    for (int i = 0; i < (L.p.a_runs ? 8 : 2) && !rc; ++i)  // 128-row boxes, 64 (half pairs), ... 1 (runs)
      rc = make_tmap(&am.m[i], L.a, (uint64_t)L.p.kdim, (uint64_t)L.a_rows, BK, BM >> i);
    if (!rc && !L.p.a_runs) memcpy(&am.m[2], &am.m[0], 6 * sizeof(CUtensorMap));  // unused
  }
  if (rc) return rc;
  rc = make_tmap(&tb, L.b, (uint64_t)L.p.kdim, (uint64_t)(L.p.a_shards ? 1 : L.p.E_l) * L.p.n_total, BK, C::B_ROWS);
  if (rc) return rc;
  if (int arc = smem_attr(reinterpret_cast<const void*>(grouped_gemm_kernel<CG, MAXE, QD>), C::SMEM)) return arc;
  int grid = L.grid > 0 ? L.grid : num_sms();
  if (const char* g = getenv("MSI_GEMM_GRID")) {  // A/B: persistent grid on fewer SMs
    const int v = atoi(g);
    if (v >= CG && v < grid) grid = v;
  }
  constexpr int kCluster = QD ? 4 : CG;
  grid -= grid % kCluster;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attrs[2];
  int na = 0;
  if (CG == 2) {
    attrs[na].id = cudaLaunchAttributeClusterDimension;
    attrs[na].val.clusterDim.x = kCluster;
    attrs[na].val.clusterDim.y = 1;
    attrs[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl_enabled()) {  // programmatic dependent launch (common.cuh)
    attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attrs;
  cfg.numAttrs = na;
  GemmParams prm = L.p;
  prm.a64 = half_pair_box64();
  prm.l2hint = l2_hints();
  {
    const char* v = getenv("MSI_GEMM_PFB");
    prm.pfb = v ? atoi(v) : 0;
  }
  MSI_CUDA(cudaLaunchKernelEx(&cfg, grouped_gemm_kernel<CG, MAXE, QD>, am, tb, prm));
  return check_launch("grouped_gemm_kernel");
}

// CTA-group selection: MSI_GEMM_CG=1|2 (or msi_set_gemm_cta_group) overrides;
// default = CTA pairs (see default_cg).
static int g_cg_override = 0;

int default_cg() {
  if (g_cg_override) return g_cg_override;
  static int cg = 0;
  if (!cg) {
    // CTA pairs by default: 4-17 % faster than 1-CTA tiles for t_e <= 1024
    // (interleaved A/B, profiles/r01_gemm_ab.jsonl), 2-3 % slower at 1536
    const char* v = getenv("MSI_GEMM_CG");
    cg = (v && v[0] == '1') ? 1 : 2;
  }
  return cg;
}

// Quad clusters (two CTA pairs sharing A by multicast): MSI_GEMM_QUAD=1
bool quad_enabled() {
  const char* v = getenv("MSI_GEMM_QUAD");
  return v && v[0] == '1';
}

int grouped_gemm_launch(const GemmLaunch& L, cudaStream_t st) {
  MSI_REQUIRE(L.p.tile_ctr != nullptr, "grouped_gemm: tile counter required");
  MSI_REQUIRE(L.p.E_l >= 1 && L.p.E_l <= MSI_MAX_LOCAL_EXPERTS, "grouped_gemm: E_l out of range");
  MSI_REQUIRE(L.p.kdim % BK == 0 && L.p.n_total % BN == 0, "grouped_gemm: K %% 64 and N %% 256 required");
  const int cg = L.cta_group ? L.cta_group : default_cg();
  if (cg == 2 && L.p.E_l <= MSI_SMALL_LOCAL_EXPERTS && quad_enabled() && L.p.nt % 2 == 0 && !L.p.a_runs &&
      !L.p.a_shards && L.p.ksplit <= 1 && !l2_hints() && half_pair_box64())
    return launch_cg<2, MSI_SMALL_LOCAL_EXPERTS, true>(L, st);
  if (L.p.E_l > MSI_SMALL_LOCAL_EXPERTS)
    return cg == 1 ? launch_cg<1, MSI_MAX_LOCAL_EXPERTS>(L, st) : launch_cg<2, MSI_MAX_LOCAL_EXPERTS>(L, st);
  return cg == 1 ? launch_cg<1, MSI_SMALL_LOCAL_EXPERTS>(L, st) : launch_cg<2, MSI_SMALL_LOCAL_EXPERTS>(L, st);
}

int pack_w13(const void* gate, const void* up, void* out, int E_l, int inter, int hidden, cudaStream_t st) {
  MSI_REQUIRE(inter % 128 == 0 && hidden % 8 == 0, "pack_w13: inter %% 128 and hidden %% 8 required");
  pack_w13_kernel<<<4 * num_sms(), 256, 0, st>>>(reinterpret_cast<const uint4*>(gate),
                                                 reinterpret_cast<const uint4*>(up),
                                                 reinterpret_cast<uint4*>(out), E_l, inter, hidden);
  return check_launch("pack_w13_kernel");
}

// Tile counters of the context-free msi_grouped_ffn, one pair per device
// (allocated zeroed on first use; each launch leaves its counter at 0).
// Calls on one device are therefore serialised on a stream by the caller.
static uint32_t* local_tile_counters(int* rc) {
  static uint32_t* ctr[64] = {};
  int dev = 0;
  *rc = (int)cudaGetDevice(&dev);
  if (*rc) return nullptr;
  if (dev < 0 || dev >= 64) { set_error("grouped_ffn: device id %d", dev); *rc = MSI_EINVAL; return nullptr; }
  if (!ctr[dev]) {
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, 256);
    if (e == cudaSuccess) e = cudaMemset(p, 0, 256);
    if (e != cudaSuccess) { set_error("grouped_ffn: tile counters: %s", cudaGetErrorString(e)); *rc = (int)e; return nullptr; }
    ctr[dev] = reinterpret_cast<uint32_t*>(p);
  }
  return ctr[dev];
}

int grouped_ffn_local(const void* x, const int32_t* total, int E_l, int rows, const void* w13,
                      const void* w2, void* hbuf, void* y, int hidden, int inter, cudaStream_t st) {
  MSI_REQUIRE(hidden % 256 == 0 && inter % 128 == 0, "grouped_ffn: hidden %% 256 and inter %% 128 required");
  int crc = 0;
  uint32_t* ctrs = local_tile_counters(&crc);
  if (!ctrs) return crc;
  GemmLaunch g1{};
  g1.a = x;
  g1.a_rows = rows;
  g1.b = w13;
  g1.p.E_l = E_l;
  g1.p.n_total = 2 * inter;
  g1.p.nt = 2 * inter / BN;
  g1.p.kdim = hidden;
  g1.p.totals = total;
  g1.p.mode = 0;
  g1.p.out = reinterpret_cast<__nv_bfloat16*>(hbuf);
  g1.p.out_ld = inter;
  g1.p.tile_ctr = ctrs;
  int rc = grouped_gemm_launch(g1, st);
  if (rc) return rc;
  GemmLaunch g2{};
  g2.a = hbuf;
  g2.p.tile_ctr = ctrs + 32;
  g2.a_rows = rows;
  g2.b = w2;
  g2.p.E_l = E_l;
  g2.p.n_total = hidden;
  g2.p.nt = hidden / BN;
  g2.p.kdim = inter;
  g2.p.totals = total;
  g2.p.mode = 1;
  g2.p.out = reinterpret_cast<__nv_bfloat16*>(y);
  g2.p.out_ld = hidden;
  return grouped_gemm_launch(g2, st);
}

// The expert FFN on receive regions without a context (tests and A/B runs):
// x_reg holds n_src regions of cap_s rows per local expert (region (e, s) at
// row (e * n_src + s) * cap_s), cntab [n_src][E_l] uint64 whose low 32 bits
// are the rows of region (e, s).  GEMM1 reads A as region runs (a_runs = 0:
// one 128-row box per tile from the expert's first region -- only valid
// when every expert has one non-empty region), GEMM2 stores Y over X in the
// regions of y_reg (may alias x_reg).  hbuf >= rows x H' (compact per expert).
int grouped_ffn_regions(const void* x_reg, const uint64_t* cntab, int n_src, int64_t cap_s, int E_l,
                        const void* w13, const void* w2, void* hbuf, int64_t hbuf_rows, void* y_reg, int hidden,
                        int inter, int a_runs, void* xcomp, cudaStream_t st) {
  MSI_REQUIRE(hidden % 256 == 0 && inter % 128 == 0, "grouped_ffn_regions: hidden %% 256 and inter %% 128 required");
  MSI_REQUIRE(n_src >= 1 && n_src <= MSI_MAX_RANKS && cap_s >= 1, "grouped_ffn_regions: bad n_src / cap_s");
  int crc = 0;
  uint32_t* ctrs = local_tile_counters(&crc);
  if (!ctrs) return crc;
  const int64_t rows = (int64_t)E_l * n_src * cap_s;
  GemmLaunch g1{};
  g1.a = x_reg;
  g1.a_rows = rows;
  if (xcomp) {  // gather the regions into compact segments first (msi_expert_ffn's path for n_a > 1)
    int grc = gather_regions(x_reg, cntab, E_l, 0, n_src, E_l, cap_s, hidden, xcomp, nullptr, 0, nullptr, 0, 0,
                             nullptr, st);
    if (grc) return grc;
    g1.a = xcomp;
    g1.a_rows = hbuf_rows;
    a_runs = 0;
  }
  g1.b = w13;
  g1.p.E_l = E_l;
  g1.p.n_total = 2 * inter;
  g1.p.nt = 2 * inter / BN;
  g1.p.kdim = hidden;
  g1.p.cntab = cntab;
  g1.p.n_a = n_src;
  g1.p.E = E_l;
  g1.p.n_src = a_runs ? n_src : 0;
  g1.p.cap_s = cap_s;
  g1.p.a_runs = a_runs;
  g1.p.mode = 0;
  g1.p.out = reinterpret_cast<__nv_bfloat16*>(hbuf);
  g1.p.out_ld = inter;
  g1.p.tile_ctr = ctrs;
  const bool dbg = getenv("MSI_DBG_SYNC") != nullptr;  // hang bisection: sync + report after each launch
  if (dbg) { cudaStreamSynchronize(st); fprintf(stderr, "[dbg] gather/pre-GEMM1 done\n"); }
  int rc = grouped_gemm_launch(g1, st);
  if (rc) return rc;
  if (dbg) { cudaStreamSynchronize(st); fprintf(stderr, "[dbg] GEMM1 done\n"); }
  GemmLaunch g2{};
  g2.a = hbuf;
  g2.a_rows = hbuf_rows;
  g2.b = w2;
  g2.p.E_l = E_l;
  g2.p.n_total = hidden;
  g2.p.nt = hidden / BN;
  g2.p.kdim = inter;
  g2.p.cntab = cntab;
  g2.p.n_a = n_src;
  g2.p.E = E_l;
  g2.p.n_src = n_src;
  g2.p.cap_s = cap_s;
  g2.p.mode = 1;
  g2.p.out = reinterpret_cast<__nv_bfloat16*>(y_reg);
  g2.p.out_ld = hidden;
  g2.p.tile_ctr = ctrs + 32;
  return grouped_gemm_launch(g2, st);
}

// Dense GEMM of the attention stage on the same kernel: one "expert" of
// `rows` compact rows (E_l = 1, no count table).  tile_ctr: the caller's
// zeroed counter word (each launch leaves it at 0).
static GemmLaunch dense_launch(const void* a, int64_t rows, const void* b, int n, int k, uint32_t* tile_ctr) {
  GemmLaunch g{};
  g.a = a;
  g.a_rows = rows;
  g.b = b;
  g.p.E_l = 1;
  g.p.n_total = n;
  g.p.nt = n / BN;
  g.p.kdim = k;
  g.p.dense_rows = rows;
  g.p.mode = 1;
  g.p.tile_ctr = tile_ctr;
  return g;
}

// fp32 logits = x . wg^T on the tensor cores (the router's candidate pass,
// router.cu): E % 256 == 0, H % 64 == 0; out [rows][E] fp32.
int dense_logits_f32(const void* x, int64_t rows, const void* wg, int E, int H, float* out, uint32_t* tile_ctr,
                     cudaStream_t st, int ksplit) {
  MSI_REQUIRE(E % BN == 0 && H % BK == 0 && rows >= 0, "dense_logits: E %% 256 and H %% 64 required");
  MSI_REQUIRE(ksplit >= 1 && (H / BK) % ksplit == 0, "dense_logits: ksplit must divide H / 64");
  if (rows == 0) return 0;
  GemmLaunch g = dense_launch(x, rows, wg, E, H, tile_ctr);
  g.p.mode = 4;
  g.p.out = reinterpret_cast<__nv_bfloat16*>(out);
  g.p.out_ld = E;
  g.p.ksplit = ksplit;
  g.p.plane = (long long)rows * E;
  return grouped_gemm_launch(g, st);
}

int dense_gemm(const void* a, int64_t rows, const void* b, int n, int k, void* out, int64_t out_ld,
               const void* resid, int64_t resid_ld, uint32_t* tile_ctr, cudaStream_t st) {
  MSI_REQUIRE(rows >= 0 && rows < (1ll << 31), "dense_gemm: rows out of range");
  if (rows == 0) return 0;
  MSI_REQUIRE(a && b && out && tile_ctr, "dense_gemm: null pointer");
  MSI_REQUIRE(n > 0 && n % BN == 0 && k > 0 && k % BK == 0, "dense_gemm: N %% 256 and K %% 64 required");
  MSI_REQUIRE(out_ld >= n && out_ld % 8 == 0, "dense_gemm: out_ld must be >= N and a multiple of 8");
  MSI_REQUIRE(!resid || (resid_ld >= n && resid_ld % 8 == 0), "dense_gemm: resid_ld must be >= N and a multiple of 8");
  if (rows == 0) return 0;
  GemmLaunch g = dense_launch(a, rows, b, n, k, tile_ctr);
  g.p.out = reinterpret_cast<__nv_bfloat16*>(out);
  g.p.out_ld = (int)out_ld;
  g.p.resid = reinterpret_cast<const __nv_bfloat16*>(resid);
  g.p.resid_ld = resid_ld;
  return grouped_gemm_launch(g, st);
}

int qkv_rope_append(const void* x, int64_t rows, int hidden, const void* wqkv, int n_heads, int n_kv,
                    const int32_t* pos, float theta, const int32_t* block_table, int max_pages, void* k_cache,
                    void* v_cache, void* q_out, uint32_t* tile_ctr, cudaStream_t st) {
  MSI_REQUIRE(rows >= 0 && rows < (1ll << 31), "qkv_rope_append: rows out of range");
  if (rows == 0) return 0;
  MSI_REQUIRE(x && wqkv && pos && block_table && k_cache && v_cache && q_out && tile_ctr,
              "qkv_rope_append: null pointer");
  MSI_REQUIRE(n_kv > 0 && n_heads > 0 && n_heads % n_kv == 0, "qkv_rope_append: bad head counts");
  const int n = (n_heads + 2 * n_kv) * MSI_HEAD_DIM;
  MSI_REQUIRE(n % BN == 0, "qkv_rope_append: n_heads + 2 n_kv must be even (256-column N tiles)");
  MSI_REQUIRE(hidden > 0 && hidden % BK == 0, "qkv_rope_append: hidden %% 64 required");
  MSI_REQUIRE(theta > 0.f && max_pages > 0, "qkv_rope_append: bad theta / max_pages");
  const RopeInv rope = rope_inv_table(theta);
  if (rows == 0) return 0;
  GemmLaunch g = dense_launch(x, rows, wqkv, n, hidden, tile_ctr);
  g.p.mode = 2;
  g.p.pos = pos;
  g.p.rope = rope;
  g.p.block_table = block_table;
  g.p.max_pages = max_pages;
  g.p.n_heads = n_heads;
  g.p.n_kv = n_kv;
  g.p.q_out = reinterpret_cast<__nv_bfloat16*>(q_out);
  g.p.k_cache = reinterpret_cast<__nv_bfloat16*>(k_cache);
  g.p.v_cache = reinterpret_cast<__nv_bfloat16*>(v_cache);
  return grouped_gemm_launch(g, st);
}

}  // namespace msi

#if MSI_GEMM_PROF
// read and reset the MMA-issuer wait profile (diagnostic builds only)
extern "C" int msi_dbg_gemm_prof(unsigned long long* out) {
  if (cudaMemcpyFromSymbol(out, msi::g_gemm_prof, sizeof(msi::g_gemm_prof)) != cudaSuccess) return -1;
  const unsigned long long z[4] = {0, 0, 0, 0};
  return cudaMemcpyToSymbol(msi::g_gemm_prof, z, sizeof(z)) == cudaSuccess ? 0 : -1;
}
#endif

extern "C" int msi_grouped_ffn_regions(const void* x_reg, const uint64_t* cntab, int n_src, int64_t cap_s, int E_l,
                                       const void* w13, const void* w2, void* hbuf, int64_t hbuf_rows, void* y_reg,
                                       int hidden, int inter, int a_runs, void* xcomp, void* stream) {
  return msi::grouped_ffn_regions(x_reg, cntab, n_src, cap_s, E_l, w13, w2, hbuf, hbuf_rows, y_reg, hidden, inter,
                                  a_runs, xcomp, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int msi_dense_logits(const void* x, int64_t T, const void* wg, int E, int H, float* out, uint32_t* tile_ctr,
                                void* stream) {
  MSI_REQUIRE(T == 0 || (x && wg && out && tile_ctr), "msi_dense_logits: null pointer");
  return msi::dense_logits_f32(x, T, wg, E, H, out, tile_ctr, reinterpret_cast<cudaStream_t>(stream), 1);
}

extern "C" int msi_dense_gemm(const void* a, int64_t rows, const void* b, int n, int k, void* out, int64_t out_ld,
                              const void* resid, int64_t resid_ld, uint32_t* tile_ctr, void* stream) {
  return msi::dense_gemm(a, rows, b, n, k, out, out_ld, resid, resid_ld, tile_ctr,
                         reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int msi_qkv_rope_append(const void* x, int64_t T, int hidden, const void* wqkv, int n_heads, int n_kv,
                                   const int32_t* pos, float theta, const int32_t* block_table, int max_pages,
                                   void* k_cache, void* v_cache, void* q_out, uint32_t* tile_ctr, void* stream) {
  return msi::qkv_rope_append(x, T, hidden, wqkv, n_heads, n_kv, pos, theta, block_table, max_pages, k_cache,
                              v_cache, q_out, tile_ctr, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int msi_pack_w13(const void* w_gate, const void* w_up, void* w13, int E_l, int inter,
                            int hidden, void* stream) {
  return msi::pack_w13(w_gate, w_up, w13, E_l, inter, hidden, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int msi_grouped_ffn(const void* x, const int32_t* total, int E_l, int rows, const void* w13,
                               const void* w2, void* hbuf, void* y, int hidden, int inter, void* stream) {
  return msi::grouped_ffn_local(x, total, E_l, rows, w13, w2, hbuf, y, hidden, inter,
                                reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int msi_set_gemm_cta_group(int cg) {
  MSI_REQUIRE(cg == 0 || cg == 1 || cg == 2, "msi_set_gemm_cta_group: 0 (default), 1 or 2");
  msi::g_cg_override = cg;
  return 0;
}
