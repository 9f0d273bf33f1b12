// router.cu -- fused gate GEMM + top-K + normalized weights + per-expert
// counts + slot placement, optionally fused
// with the M2N dispatch of the routed rows (route.h).
//
// One kernel launch (fine-grained MoE at small T: a logits kernel on a
// token x expert grid, then route_kernel for phases 2-5).  Each CTA takes a
// virtual block id (atomic ticket: every lower block has started) and owns BT
// consecutive tokens:
//   1. logits[t,e] in the pinned fp32 order (lane l accumulates elements
//      256j + 8l + c with fmaf, then an xor butterfly 16,8,4,2,1) -- the
//      order oracle/msi_oracle.c restates, so routing is bit-exact;
//   2. top-K per token (warp arg-max, ties to the lower expert), weights =
//      softmax of the K chosen logits with det_expf (bit-exact as well);
//   3. in-CTA ranks (BT <= 32 tokens, one warp): bit `lane` of mask[p] marks
//      "token lane chose p", so rank = popc(mask[p] & lanes_below);
//   4. decoupled look-back: the CTA publishes its per-slot histogram, sums the
//      histograms (or the first inclusive prefix) of the blocks before it, and
//      publishes its inclusive prefix -- every CTA gets its slot bases without
//      a second pass or a serial last-CTA scan;
//   5. (dispatch) the CTA's rows go straight to the expert GPUs' receive
//      regions (16-B stores over NVLink peer memory); the last CTA to finish
//      publishes the sender's counts and releases the arrival counters.
// HBM-bound for small E (x read once; the dispatch re-reads the CTA's rows from
// L2); FMA-bound for E = 256 (logits on CUDA cores because the fixed reduction
// order is the bit-exactness contract).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "gemm.h"
#include "route.h"

namespace msi {

int num_sms();  // expert_gemm.cu

namespace {

constexpr int kWarps = 8;

// Packed fp32x2 FMAs in the logits loop (compile with -DMSI_ROUTER_FFMA2=0 for
// the scalar-FFMA build; both are bit-identical)
#ifndef MSI_ROUTER_FFMA2
#define MSI_ROUTER_FFMA2 1
#endif
#ifndef MSI_EXACT_U  // route_tc candidate pass: 256-element chunks loaded ahead per warp
#define MSI_EXACT_U 4
#endif
#ifndef MSI_ROUTE_LB  // route_kernel min CTAs per SM (register budget)
#define MSI_ROUTE_LB 2
#endif
#ifndef MSI_ROUTER_EP
#define MSI_ROUTER_EP 1
#endif
#ifndef MSI_DISP_U
#define MSI_DISP_U 12  // measured 73-74 -> 71 us at T = 3072, E = 8 (scripts/r02_ab_dispu.sh)
#endif
constexpr uint32_t kTaken = 0x7fc0dead;  // NaN payload marking an already-selected expert

// Shared memory: logits [max(BT,16)][E] fp32 (reused after top-K for the [P]
// slot masks and [P] bases), then -- when WS -- a copy of W_g [E][H] bf16 so
// the FMA loop reads the gate weights at shared-memory latency.
__host__ __device__ inline size_t logit_smem_bytes(int BT, int E) {
  return (size_t)(BT > 16 ? BT : 16) * E * sizeof(float) + (size_t)E * sizeof(uint32_t);
}

// shared memory before the staged W_g: logits, or the [P] masks + [P] bases
__host__ __device__ inline size_t tail_smem_bytes(int BT, int E, int P) {
  size_t head = logit_smem_bytes(BT, E);
  if (head < (size_t)P * 8) head = (size_t)P * 8;
  return (head + 15) & ~size_t(15);
}

// Replicated-expert placement: rep[e*(R+1)] = number of
// replicas of logical expert e, rep[e*(R+1)+1+r] = physical slot of replica r.
// Token t of sender s routed to e goes to replica (t + s) mod nrep[e]; counts
// and slots are then per physical slot (P of them).  rep == nullptr: P = E,
// physical = logical.
struct Placement {
  const int32_t* rep;
  int R, P, sender;
  int32_t* pidx;  // [T,K] physical slot per (t,k) (may alias idx when rep == nullptr)
  int pfw;        // 1 = prefetch the next W_g chunk into L1 (MSI_ROUTER_PFW, unstaged W_g only)
};

// Workspace: [0] finish ticket, [1] virtual-block ticket (both back to 0 at the
// end of every launch), u64 at byte 64 = launch generation, u64 look-back
// words [nblk][P] from byte 128: (generation << 32 | flag << 30 | count).
constexpr size_t kLbOffset = 128;
constexpr uint32_t kAgg = 1u, kInc = 2u;

__device__ __forceinline__ uint64_t lb_word(uint32_t gen, uint32_t flag, uint32_t v) {
  return ((uint64_t)gen << 32) | ((uint64_t)flag << 30) | (uint64_t)v;
}
__device__ __forceinline__ void st_volatile64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_volatile64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Virtual block id and launch generation of this CTA (thread 0 takes them).
struct BlockId {
  int vb;
  uint32_t gen;
};
__device__ __forceinline__ BlockId take_block(int32_t* ws) {
  __shared__ int s_vb;
  __shared__ uint32_t s_gen;
  if (threadIdx.x == 0) {
    s_vb = atomicAdd(&ws[1], 1);
    s_gen = (uint32_t)(*reinterpret_cast<volatile uint64_t*>(ws + 16)) + 1u;
  }
  __syncthreads();
  return BlockId{s_vb, s_gen};
}

// Phases 2-5 (shared by both logit kernels): s_logit [BT][E] holds this CTA's
// logits; produces idx, w (and pidx), the final slots, the counts (the last
// virtual block) and, with d.on, the dispatch of the CTA's rows.
__device__ __forceinline__ void route_tail(const __nv_bfloat16* __restrict__ x, float* s_logit, BlockId b, int nblk,
                                           int BT, int T, int E, int K, int32_t* __restrict__ idx_out,
                                           float* __restrict__ w_out, int32_t* __restrict__ cnt_out,
                                           int32_t* __restrict__ slot_out, int32_t* __restrict__ ws,
                                           const Placement& pl, const DispatchArgs& d) {
  __shared__ int s_last;
  __shared__ uint32_t s_epoch;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t0 = b.vb * BT;
  if (d.on && b.vb == 0 && threadIdx.x == 0) trace_stamp(d.trace, 0);
  // ---- 2. top-K + weights (one warp per token) ----------------------------
  for (int lt = warp; lt < BT; lt += kWarps) {
    const int t = t0 + lt;
    if (t >= T) break;
    float* lg = s_logit + lt * E;
    float selv[32];
    int seli[32];
    for (int k = 0; k < K; ++k) {
      float bv = -INFINITY;
      int bi = 0x7fffffff;
      for (int e = lane; e < E; e += 32) {
        float v = lg[e];
        if (__float_as_uint(v) == kTaken) continue;
        if (v > bv || (v == bv && e < bi)) { bv = v; bi = e; }
      }
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) {
        float ov = __shfl_xor_sync(0xffffffffu, bv, off);
        int oi = __shfl_xor_sync(0xffffffffu, bi, off);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
      }
      selv[k] = bv;
      seli[k] = bi;
      __syncwarp();
      if (lane == 0) lg[bi] = __uint_as_float(kTaken);  // exclude from later rounds
      __syncwarp();
    }
    if (lane == 0) {
      float ex[32], s = 0.0f;
      for (int k = 0; k < K; ++k) {
        ex[k] = det_expf(__fsub_rn(selv[k], selv[0]));
        s = (k == 0) ? ex[0] : __fadd_rn(s, ex[k]);
      }
      for (int k = 0; k < K; ++k) {
        idx_out[(size_t)t * K + k] = seli[k];
        w_out[(size_t)t * K + k] = __fdiv_rn(ex[k], s);
        if (pl.rep) {
          const int32_t* re = pl.rep + (size_t)seli[k] * (pl.R + 1);
          pl.pidx[(size_t)t * K + k] = re[1 + (t + pl.sender) % re[0]];
        }
      }
    }
  }
  __syncthreads();

  // ---- 3. in-CTA ranks (BT <= 32 tokens = one warp chunk): lane = token,
  //      bit `lane` of mask[p] says "this token chose physical slot p"
  const int P = pl.P;
  const int32_t* pidx = pl.rep ? pl.pidx : idx_out;
  uint32_t* mask = reinterpret_cast<uint32_t*>(s_logit);  // [P] (logits no longer needed)
  int32_t* s_base = reinterpret_cast<int32_t*>(mask + P);  // [P] exclusive bases of this CTA
  for (int e = threadIdx.x; e < P; e += blockDim.x) mask[e] = 0u;
  __syncthreads();
  if (warp == 0) {
    const int t = t0 + lane;
    if (lane < BT && t < T)
      for (int k = 0; k < K; ++k) atomicOr(&mask[pidx[(size_t)t * K + k]], 1u << lane);
  }
  __syncthreads();

  // ---- 4. decoupled look-back over the virtual blocks before this one -----
  uint64_t* lb = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(ws) + kLbOffset);
  uint64_t* mine = lb + (size_t)b.vb * P;
  for (int p = threadIdx.x; p < P; p += blockDim.x)  // aggregate first (block 0: already inclusive)
    st_volatile64(mine + p, lb_word(b.gen, b.vb == 0 ? kInc : kAgg, __popc(mask[p])));
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    // walk back over the predecessors' words LB at a time: the LB loads are
    // independent (one L2 round trip per batch instead of one per block --
    // with every block arriving together only block 0 is inclusive at first,
    // and a one-at-a-time walk cost ~1 us per predecessor); a word not yet
    // published is re-polled on its own, and the sum stops at the first
    // inclusive prefix, in block order as before
    constexpr int LB = 8;
    uint32_t excl = 0;
    for (int j = b.vb - 1; j >= 0; j -= LB) {
      uint64_t v[LB];
#pragma unroll
      for (int q = 0; q < LB; ++q) v[q] = (j - q >= 0) ? ld_volatile64(lb + (size_t)(j - q) * P + p) : 0ull;
      bool inc = false;
#pragma unroll
      for (int q = 0; q < LB; ++q) {
        if (j - q < 0) break;
        while ((uint32_t)(v[q] >> 32) != b.gen) v[q] = ld_volatile64(lb + (size_t)(j - q) * P + p);
        excl += (uint32_t)v[q] & 0x3fffffffu;
        if (((uint32_t)v[q] >> 30 & 3u) == kInc) { inc = true; break; }
      }
      if (inc) break;
    }
    const uint32_t h = __popc(mask[p]);
    if (b.vb > 0) st_volatile64(mine + p, lb_word(b.gen, kInc, excl + h));
    s_base[p] = (int32_t)excl;
    if (b.vb == nblk - 1) cnt_out[p] = (int32_t)(excl + h);
  }
  __syncthreads();
  if (warp == 0) {  // final slots: rank among the sender's earlier tokens
    const int t = t0 + lane;
    const uint32_t below = (1u << lane) - 1u;
    if (lane < BT && t < T)
      for (int k = 0; k < K; ++k) {
        const int p = pidx[(size_t)t * K + k];
        slot_out[(size_t)t * K + k] = s_base[p] + __popc(mask[p] & below);
      }
  }

  // ---- 5. dispatch: this CTA's rows into the expert GPUs' receive regions --
  if (d.on) {
    if (threadIdx.x == 0) s_epoch = resolve_epoch(d.epoch, d.ause, 1u, d.status);  // 0 = mismatch: send nothing
    __syncthreads();
    if (s_epoch) {
      const size_t row_bytes = (size_t)d.H * 2;
      const int nchunk = d.H >> 8;  // 512-B warp chunks per row
      const int ndst = K * d.tp;
      for (int lt = warp; lt < BT; lt += kWarps) {
        const int t = t0 + lt;
        if (t >= T) break;
        // lane j < K*tp resolves destination j: (t, k = j / tp) on GPU r = j % tp of the node
        char* my_dst = nullptr;
        if (lane < ndst) {
          const int k = lane / d.tp, r = lane - k * d.tp;
          const int p = pidx[(size_t)t * K + k];
          const int q = (p / d.E_l) * d.tp + r;
          const long long row = d.slot_row0 + ((long long)(p % d.E_l) * d.n_send + d.s) * d.cap_s +
                                slot_out[(size_t)t * K + k];
          my_dst = d.recv[q] + row * row_bytes;
        }
        const char* src = reinterpret_cast<const char*>(x + (size_t)t * d.H) + lane * 16;
        constexpr int U = MSI_DISP_U;  // 512-B row chunks loaded per lane before the stores
        for (int j0 = 0; j0 < nchunk; j0 += U) {
          uint4 v[U];
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (j0 + u < nchunk) v[u] = ld_nc_v4(src + (size_t)(j0 + u) * 512);
          for (int j = 0; j < ndst; ++j) {
            char* dst = reinterpret_cast<char*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(my_dst), j)) +
                        lane * 16;
#pragma unroll
            for (int u = 0; u < U; ++u)
              if (j0 + u < nchunk) st_v4(dst + (size_t)(j0 + u) * 512, v[u]);
          }
        }
      }
    }
  }

  // ---- 6. the last CTA to finish: counts to the receivers, release, reset --
  __syncthreads();
  if (threadIdx.x == 0) {
    if (d.on) __threadfence_system();  // this CTA's peer row stores before the ticket
    else __threadfence();
    s_last = atomicAdd(&ws[0], 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (d.on && s_epoch) {
    // the sender's counts (the last virtual block's inclusive prefix), tagged
    // with the epoch, into every expert GPU's count table
    const uint32_t ep = s_epoch;
    for (int i = threadIdx.x; i < d.n_e * P; i += blockDim.x) {
      const int q = i / P, p = i - q * P;
      const uint32_t c = (uint32_t)ld_volatile64(lb + (size_t)(nblk - 1) * P + p) & 0x3fffffffu;
      st_relaxed_sys64(d.cntab[q] + (size_t)d.s * P + p, ((uint64_t)ep << 32) | c);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      *d.ause = ep;  // every CTA has read the old value
      trace_stamp(d.trace, 2);
      fence_sys();
      for (int q = 0; q < d.n_e; ++q) red_release_sys_add(d.arrive[q], 1u);
    }
  }
  if (threadIdx.x == 0) {
    ws[0] = 0;
    ws[1] = 0;
    *reinterpret_cast<volatile uint64_t*>(ws + 16) = b.gen;
  }
}

// Logits of one warp tile: TT tokens from t_first x TE experts from e_first.
// Lane l accumulates elements 256j + 8l + c (j ascending, c = 0..7) with
// fmaf from +0, then an xor butterfly 16,8,4,2,1 -- the pinned order
// (oracle/msi_oracle.c); every lane returns the final values, NaN as -inf.
template <int TT, int TE, bool WS, int PF = (TT * TE > 32) ? 2 : 4>
__device__ __forceinline__ void tile_logits(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ wg,
                                            int t_first, int e_first, int T, int H, float (&acc)[TT][TE],
                                            int pfw = 0) {
  const int lane = threadIdx.x & 31;
  const int nchunk = H >> 8;
#pragma unroll
  for (int i = 0; i < TT; ++i)
#pragma unroll
    for (int j = 0; j < TE; ++j) acc[i][j] = 0.0f;
  // packed FFMA2 accumulators (two experts per float2) on the unstaged path
  constexpr bool kPair = MSI_ROUTER_FFMA2 && TE % 2 == 0 && !WS;
  float2 acc2[TT][(TE + 1) / 2];
#pragma unroll
  for (int i = 0; i < TT; ++i)
#pragma unroll
    for (int j = 0; j < (TE + 1) / 2; ++j) acc2[i][j] = make_float2(0.0f, 0.0f);
  const __nv_bfloat16* xr[TT];
  bool tv[TT];
#pragma unroll
  for (int i = 0; i < TT; ++i) {
    int t = t_first + i;
    tv[i] = t < T;
    xr[i] = x + (size_t)(tv[i] ? t : 0) * H + 8 * lane;
  }
  const __nv_bfloat16* wr = wg + (size_t)e_first * H + 8 * lane;
  // x chunks are prefetched PF iterations ahead (HBM latency), W_g rows are
  // small and L1/L2-resident; the accumulation order per (token, expert)
  // stays j-major, c-minor as pinned.
  uint4 xq[PF][TT];
#pragma unroll
  for (int u = 0; u < PF; ++u)
#pragma unroll
    for (int i = 0; i < TT; ++i)
      xq[u][i] = (tv[i] && u < nchunk) ? __ldg(reinterpret_cast<const uint4*>(xr[i] + 256 * u)) : make_uint4(0, 0, 0, 0);
  for (int j0 = 0; j0 < nchunk; j0 += PF) {
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      const int j = j0 + u;
      if (j >= nchunk) break;
      // unstaged W_g: pull chunk j + 1 of the TE rows into L1 now, so the
      // loads below hit L1 instead of paying an L2 round trip per chunk (no
      // registers held; the arithmetic and its order are unchanged)
      if (!WS && pfw && j + 1 < nchunk && (lane & 7) == 0) {
#pragma unroll
        for (int e = 0; e < TE; ++e)
          asm volatile("prefetch.global.L1 [%0];" ::"l"(wr + (size_t)e * H + 256 * (j + 1)));
      }
      float xv[TT][8];
#pragma unroll
      for (int i = 0; i < TT; ++i) {
        const uint4 v = xq[u][i];
        xv[i][0] = bf16lo(v.x); xv[i][1] = bf16hi(v.x);
        xv[i][2] = bf16lo(v.y); xv[i][3] = bf16hi(v.y);
        xv[i][4] = bf16lo(v.z); xv[i][5] = bf16hi(v.z);
        xv[i][6] = bf16lo(v.w); xv[i][7] = bf16hi(v.w);
        // refill this slot with chunk j + PF
        xq[u][i] = (tv[i] && j + PF < nchunk) ? __ldg(reinterpret_cast<const uint4*>(xr[i] + 256 * (j + PF)))
                                             : make_uint4(0, 0, 0, 0);
      }
      if constexpr (kPair) {
        // two experts per packed FFMA2 (sm_100 fma.rn.f32x2): each half is
        // the same IEEE fmaf in the same c order, so the logits are
        // bit-identical to the scalar loop at half the FMA issue count.
        // FMA-bound unstaged path only: the HBM-bound staged-W_g kernels
        // (E <= 16) measured ~3 % slower with it (E = 16: 29 -> 30 us)
        // EP expert pairs interleaved per c step: independent FFMA2s between
        // two updates of one accumulator (MSI_ROUTER_EP, default 1)
        constexpr int EP = (TE % (2 * MSI_ROUTER_EP) == 0) ? MSI_ROUTER_EP : 1;
#pragma unroll
        for (int e0 = 0; e0 < TE; e0 += 2 * EP) {
          float2 w2[EP][8];
#pragma unroll
          for (int p = 0; p < EP; ++p) {
            const int e = e0 + 2 * p;
            const uint4* wp0 = reinterpret_cast<const uint4*>(wr + (size_t)e * H + 256 * j);
            const uint4* wp1 = reinterpret_cast<const uint4*>(wr + (size_t)(e + 1) * H + 256 * j);
            const uint4 v0 = WS ? *wp0 : __ldg(wp0), v1 = WS ? *wp1 : __ldg(wp1);
            w2[p][0] = make_float2(bf16lo(v0.x), bf16lo(v1.x)); w2[p][1] = make_float2(bf16hi(v0.x), bf16hi(v1.x));
            w2[p][2] = make_float2(bf16lo(v0.y), bf16lo(v1.y)); w2[p][3] = make_float2(bf16hi(v0.y), bf16hi(v1.y));
            w2[p][4] = make_float2(bf16lo(v0.z), bf16lo(v1.z)); w2[p][5] = make_float2(bf16hi(v0.z), bf16hi(v1.z));
            w2[p][6] = make_float2(bf16lo(v0.w), bf16lo(v1.w)); w2[p][7] = make_float2(bf16hi(v0.w), bf16hi(v1.w));
          }
#pragma unroll
          for (int c = 0; c < 8; ++c)
#pragma unroll
            for (int p = 0; p < EP; ++p)
#pragma unroll
              for (int i = 0; i < TT; ++i)
                acc2[i][(e0 >> 1) + p] = __ffma2_rn(make_float2(xv[i][c], xv[i][c]), w2[p][c], acc2[i][(e0 >> 1) + p]);
        }
      } else {
#pragma unroll
        for (int e = 0; e < TE; ++e) {
          const uint4* wp = reinterpret_cast<const uint4*>(wr + (size_t)e * H + 256 * j);
          uint4 v = WS ? *wp : __ldg(wp);
          float wv[8] = {bf16lo(v.x), bf16hi(v.x), bf16lo(v.y), bf16hi(v.y),
                         bf16lo(v.z), bf16hi(v.z), bf16lo(v.w), bf16hi(v.w)};
#pragma unroll
          for (int c = 0; c < 8; ++c)
#pragma unroll
            for (int i = 0; i < TT; ++i) acc[i][e] = __fmaf_rn(xv[i][c], wv[c], acc[i][e]);
        }
      }
    }
  }
  if constexpr (kPair) {
#pragma unroll
    for (int i = 0; i < TT; ++i)
#pragma unroll
      for (int e = 0; e < TE; e += 2) {
        acc[i][e] = acc2[i][e >> 1].x;
        acc[i][e + 1] = acc2[i][e >> 1].y;
      }
  }
#pragma unroll
  for (int i = 0; i < TT; ++i)
#pragma unroll
    for (int e = 0; e < TE; ++e) {
      float v = acc[i][e];
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
      acc[i][e] = (v != v) ? -INFINITY : v;  // NaN logits rank as -inf (the oracle does the same)
    }
}


// Fine-grained MoE (E >= 64, FMA-bound): the logits get their own 2-D grid --
// CTA (blockIdx.x, blockIdx.y) = BT tokens x EB experts, one TT x TE warp
// tile per warp at a time, <= 128 registers so 2 CTAs share an SM -- into a
// [T][E] fp32 scratch; route_kernel then runs phases 2-5 on 32-token blocks.
// Same per-(token, expert) reduction order as the fused kernel: bit-identical.
template <int TT, int TE>
__global__ void __launch_bounds__(kWarps * 32, 2)
gate_logits_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ wg, int T, int H, int E,
                   int BT, int EB, float* __restrict__ logits, int pfw) {
  pdl_trigger();
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t0 = blockIdx.x * BT, e0 = blockIdx.y * EB;
  const int tgroups = BT / TT, egroups = EB / TE;
  for (int tile = warp; tile < tgroups * egroups; tile += kWarps) {
    const int tg = tile % tgroups, eg = tile / tgroups;
    float acc[TT][TE];
    tile_logits<TT, TE, false, (TT * TE >= 32 ? 2 : 4)>(x, wg, t0 + tg * TT, e0 + eg * TE, T, H, acc, pfw);
#pragma unroll
    for (int i = 0; i < TT; ++i) {
      const int t = t0 + tg * TT + i;
#pragma unroll
      for (int e = 0; e < TE; ++e)
        if (lane == ((i * TE + e) & 31) && t < T) logits[(size_t)t * E + e0 + eg * TE + e] = acc[i][e];
    }
  }
}

// Exact (pinned-order) logits of token row xr against up to 4 experts
// ex[0..n) -- the per-lane accumulation of tile_logits (elements 256j + 8l + c,
// j ascending, c = 0..7, fmaf from +0), then the same xor butterfly: the
// values are bit-identical to the CUDA-core logits kernels'.  Warp-collective.
__device__ __noinline__ void exact_logits4(const __nv_bfloat16* __restrict__ xr, const __nv_bfloat16* __restrict__ wg,
                                           int H, const int (&ex)[4], int n, float (&out)[4]) {
  const int lane = threadIdx.x & 31;
  float2 acc2[2] = {make_float2(0.0f, 0.0f), make_float2(0.0f, 0.0f)};  // candidates (0,1), (2,3)
  const int nchunk = H >> 8;
  const __nv_bfloat16* wq[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) wq[q] = wg + (size_t)ex[q < n ? q : 0] * H + 8 * lane;
  constexpr int U = MSI_EXACT_U;  // chunks whose loads are all issued before the FMAs (L2 latency)
  for (int j0 = 0; j0 < nchunk; j0 += U) {
    uint4 xv4[U], wv4[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool ok = j0 + u < nchunk;
      xv4[u] = ok ? __ldg(reinterpret_cast<const uint4*>(xr + 256 * (j0 + u) + 8 * lane)) : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        wv4[u][q] = (ok && q < n) ? __ldg(reinterpret_cast<const uint4*>(wq[q] + 256 * (j0 + u))) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (j0 + u >= nchunk) break;
      const uint4 xa = xv4[u];
      const float xv[8] = {bf16lo(xa.x), bf16hi(xa.x), bf16lo(xa.y), bf16hi(xa.y),
                           bf16lo(xa.z), bf16hi(xa.z), bf16lo(xa.w), bf16hi(xa.w)};
      // candidate pairs on packed FFMA2 (sm_100 fma.rn.f32x2): each half is
      // the same IEEE fmaf in the same c order as the scalar loop, at half the
      // FMA issue count; the weights' lo halves of pair 0 convert on the FMA
      // pipe, the rest on the ALU pipe (the two pipes then carry about the
      // same count; B300_MICROARCH.md pipe rates)
#pragma unroll
      for (int pr = 0; pr < 2; ++pr) {
        const uint4 v0 = wv4[u][2 * pr], v1 = wv4[u][2 * pr + 1];
        const uint32_t a0[4] = {v0.x, v0.y, v0.z, v0.w}, a1[4] = {v1.x, v1.y, v1.z, v1.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const float2 wlo = pr == 0 ? make_float2(bf16lo(a0[h]), bf16lo(a1[h]))
                                     : make_float2(bf16lo_alu(a0[h]), bf16lo_alu(a1[h]));
          const float2 whi = make_float2(bf16hi(a0[h]), bf16hi(a1[h]));
          acc2[pr] = __ffma2_rn(make_float2(xv[2 * h], xv[2 * h]), wlo, acc2[pr]);  // q >= n: unused
          acc2[pr] = __ffma2_rn(make_float2(xv[2 * h + 1], xv[2 * h + 1]), whi, acc2[pr]);
        }
      }
    }
  }
  const float acc[4] = {acc2[0].x, acc2[0].y, acc2[1].x, acc2[1].y};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    float v = acc[q];
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
    out[q] = (v != v) ? -INFINITY : v;
  }
}

// Tensor-core candidate pass (route_tc): s_logit holds logits computed on
// the tensor cores (fp32 accumulation in the MMA's order).  For every token:
// |tc - pinned| <= eps_e = c ||x_t|| ||w_e|| (c = 4 H 2^-24, a margin over
// the worst-case fp32 summation bound of both orders), so with theta = the
// K-th largest of (tc_e - eps_e) only experts with tc_e + eps_e >= theta can
// be in the pinned top-K.  Those candidates get their logits recomputed in
// the pinned order (bit-identical), every other expert -inf; non-finite
// norms or bounds recompute all E.  Top-K, weights and placement then run
// unchanged on exact values.
// Two phases so that the recompute is balanced across the CTA's warps (the
// candidate count varies per token, ~9-30 at the DS-V3 shape): A) one warp
// per token computes the bounds and writes the token's candidate list to
// s_cand; B) the CTA's (token, quad of candidates) items are dealt round-robin
// to the warps.  Each value is still one warp's pinned-order dot product.
template <int EPL>  // experts per lane (E <= 32 * EPL)
__device__ void exactify(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ wg,
                         const float* __restrict__ wnorm, float* s_logit, uint16_t* s_cand, int* s_nc, int t0,
                         int rows, int E, int K, int H) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float cb = 4.0f * (float)H * 5.9604645e-8f * 1.01f;
  for (int lt = warp; lt < rows; lt += kWarps) {
    const __nv_bfloat16* xr = x + (size_t)(t0 + lt) * H;
    float* lg = s_logit + (size_t)lt * E;
    float ss = 0.0f;
    for (int i0 = 8 * lane; i0 < H; i0 += 256 * 4) {
      uint4 v4[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        v4[u] = i0 + 256 * u < H ? __ldg(reinterpret_cast<const uint4*>(xr + i0 + 256 * u)) : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint4 v = v4[u];
        const float f[8] = {bf16lo_alu(v.x), bf16hi(v.x), bf16lo_alu(v.y), bf16hi(v.y),
                            bf16lo_alu(v.z), bf16hi(v.z), bf16lo_alu(v.w), bf16hi(v.w)};
#pragma unroll
        for (int c = 0; c < 8; ++c) ss = fmaf(f[c], f[c], ss);
      }
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    const float xn = sqrtf(ss) * 1.001f;
    float lo[EPL], hi[EPL];
    bool finite = isfinite(xn);
#pragma unroll
    for (int q = 0; q < EPL; ++q) {
      const int e = lane + 32 * q;
      if (e < E) {
        const float a = lg[e], eps = cb * xn * wnorm[e];
        lo[q] = a - eps;
        hi[q] = a + eps;
        finite &= isfinite(lo[q]) && isfinite(hi[q]);
      } else {
        lo[q] = -INFINITY;
        hi[q] = -INFINITY;
      }
    }
    finite = __all_sync(0xffffffffu, finite);
    float theta = -INFINITY;
    if (finite) {  // K-th largest lower bound: K rounds of a warp max (one removal per round)
      float cur[EPL];
#pragma unroll
      for (int q = 0; q < EPL; ++q) cur[q] = lo[q];
      for (int k = 0; k < K; ++k) {
        float bv = -INFINITY;
        int bq = -1;
#pragma unroll
        for (int q = 0; q < EPL; ++q)
          if (cur[q] > bv) { bv = cur[q]; bq = q; }
        float mv = bv;
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) mv = fmaxf(mv, __shfl_xor_sync(0xffffffffu, mv, off));
        const unsigned own = __ballot_sync(0xffffffffu, bv == mv && bq >= 0);
        if (lane == __ffs(own) - 1) cur[bq] = -INFINITY;  // remove one instance
        theta = mv;
      }
    }
    // candidate masks (bit l of mask[q]: expert l + 32 q), non-candidates -inf
    unsigned mask[EPL];
#pragma unroll
    for (int q = 0; q < EPL; ++q) {
      const bool cand = (lane + 32 * q < E) && (!finite || hi[q] >= theta);
      mask[q] = __ballot_sync(0xffffffffu, cand);
      if (!cand && lane + 32 * q < E) lg[lane + 32 * q] = -INFINITY;
    }
    // the token's candidate list, ascending expert id
    int base = 0;
#pragma unroll
    for (int q = 0; q < EPL; ++q) {
      if ((mask[q] >> lane) & 1u) s_cand[lt * E + base + __popc(mask[q] & ((1u << lane) - 1u))] = (uint16_t)(lane + 32 * q);
      base += __popc(mask[q]);
    }
    if (lane == 0) s_nc[lt] = base;
  }
  __syncthreads();
  // B: exact logits of item (token lt, candidates 4 qi .. 4 qi + 3); one call
  // site of exact_logits4 (instruction cache)
  int lt = 0, before = 0;  // items before token lt
  for (int it = warp;; it += kWarps) {
    while (lt < rows && it >= before + ((s_nc[lt] + 3) >> 2)) before += (s_nc[lt++] + 3) >> 2;
    if (lt >= rows) break;
    const int c0 = 4 * (it - before), n = min(4, s_nc[lt] - c0);
    int ex[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) ex[i] = i < n ? (int)s_cand[lt * E + c0 + i] : 0;
    float v[4];
    exact_logits4(x + (size_t)(t0 + lt) * H, wg, H, ex, n, v);
    float* lg = s_logit + (size_t)lt * E;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (i < n && lane == i) lg[ex[i]] = v[i];
  }
}

template <int EPL>
__global__ void __launch_bounds__(kWarps * 32, MSI_ROUTE_LB)
route_kernel(const __nv_bfloat16* __restrict__ x, const float* __restrict__ logits, int T, int E, int K, int BT,
             int32_t* __restrict__ idx_out, float* __restrict__ w_out, int32_t* __restrict__ cnt_out,
             int32_t* __restrict__ slot_out, int32_t* __restrict__ ws, const Placement pl, const DispatchArgs d,
             const __nv_bfloat16* __restrict__ wg, const float* __restrict__ wnorm, int H, int ksplit) {
  extern __shared__ __align__(16) float s_logit[];  // [BT][E]
  pdl_trigger();
  pdl_wait();
  const BlockId b = take_block(ws);
  const int t0 = b.vb * BT;
  const int rows = max(0, min(BT, T - t0));
  const float4* src = reinterpret_cast<const float4*>(logits + (size_t)t0 * E);
  float4* dst = reinterpret_cast<float4*>(s_logit);
  const size_t plane4 = (size_t)T * E / 4;  // split-K planes of the tensor-core logits, summed here
  for (int i = threadIdx.x; i < rows * E / 4; i += blockDim.x) {
    float4 v = __ldcg(src + i);
    for (int sp = 1; sp < ksplit; ++sp) {
      const float4 u = __ldcg(src + sp * plane4 + i);
      v.x += u.x; v.y += u.y; v.z += u.z; v.w += u.w;
    }
    dst[i] = v;
  }
  __syncthreads();
  if (wnorm) {  // tensor-core logits: exact values for the candidates
    // candidate lists after the tail's region (route_tc sizes the launch's smem)
    uint16_t* s_cand = reinterpret_cast<uint16_t*>(reinterpret_cast<char*>(s_logit) + tail_smem_bytes(BT, E, pl.P));
    int* s_nc = reinterpret_cast<int*>(s_cand + ((BT * E + 7) & ~7));
    exactify<EPL>(x, wg, wnorm, s_logit, s_cand, s_nc, t0, rows, E, K, H);
    __syncthreads();
  }
  route_tail(x, s_logit, b, (int)gridDim.x, BT, T, E, K, idx_out, w_out, cnt_out, slot_out, ws, pl, d);
}

// ||w_e||_2 per expert (rounded up) for the candidate bound of route_tc.
__global__ void __launch_bounds__(256) wg_norm_kernel(const __nv_bfloat16* __restrict__ wg, int H, float* wnorm) {
  __shared__ float s[8];
  const __nv_bfloat16* w = wg + (size_t)blockIdx.x * H;
  float ss = 0.0f;
  for (int i = 8 * threadIdx.x; i < H; i += 8 * blockDim.x) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(w + i));
    const float f[8] = {bf16lo(v.x), bf16hi(v.x), bf16lo(v.y), bf16hi(v.y),
                        bf16lo(v.z), bf16hi(v.z), bf16lo(v.w), bf16hi(v.w)};
#pragma unroll
    for (int c = 0; c < 8; ++c) ss = fmaf(f[c], f[c], ss);
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.0f;
    for (int i = 0; i < 8; ++i) t += s[i];
    wnorm[blockIdx.x] = sqrtf(t) * 1.001f;
  }
}

// Small warp tiles (TT * TE <= 16) are capped at 128 registers so two CTAs
// share an SM (16 warps; the staged W_g of E <= 16 fits twice in smem).
template <int TT, int TE, bool WS>
__global__ void __launch_bounds__(kWarps * 32, (TT * TE <= 16) ? 2 : 1)
gate_topk_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ wg,
                 int T, int H, int E, int K, int BT, int32_t* __restrict__ idx_out,
                 float* __restrict__ w_out, int32_t* __restrict__ cnt_out,
                 int32_t* __restrict__ slot_out, int32_t* __restrict__ ws, const Placement pl,
                 const DispatchArgs d) {
  extern __shared__ __align__(16) float s_logit[];         // [BT][E]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_trigger();
  pdl_wait();
  const BlockId b = take_block(ws);
  const int t0 = b.vb * BT;
  const __nv_bfloat16* wgs = wg;
  if (WS) {  // stage W_g (E*H*2 bytes) with one TMA bulk copy
    __shared__ __align__(8) uint64_t s_bar;
    char* dst = reinterpret_cast<char*>(s_logit) + ((logit_smem_bytes(BT, E) + 15) & ~size_t(15));
    const uint32_t bytes = (uint32_t)E * H * 2;
    if (threadIdx.x == 0) {
      mbar_init(&s_bar, 1);
      fence_barrier_init();
      mbar_expect_tx(&s_bar, bytes);
      bulk_g2s(dst, wg, bytes, &s_bar);
    }
    __syncthreads();
    mbar_wait(&s_bar, 0);
    wgs = reinterpret_cast<const __nv_bfloat16*>(dst);
  }

  // ---- 1. logits ---------------------------------------------------------
  const int tgroups = BT / TT, egroups = E / TE;
  for (int tile = warp; tile < tgroups * egroups; tile += kWarps) {
    const int tg = tile % tgroups, eg = tile / tgroups;
    float acc[TT][TE];
    tile_logits<TT, TE, WS>(x, wgs, t0 + tg * TT, eg * TE, T, H, acc, pl.pfw);
#pragma unroll
    for (int i = 0; i < TT; ++i)
#pragma unroll
      for (int e = 0; e < TE; ++e)
        if (lane == ((i * TE + e) & 31)) s_logit[(tg * TT + i) * E + eg * TE + e] = acc[i][e];
  }
  __syncthreads();

  route_tail(x, s_logit, b, (int)gridDim.x, BT, T, E, K, idx_out, w_out, cnt_out, slot_out, ws, pl, d);
}

constexpr size_t kMaxStagedW = 200 * 1024;  // W_g staged in smem up to this size


template <int TT, int TE>
int launch(const void* x, const void* wg, int T, int H, int E, int K, int BT, int32_t* idx,
           float* w, int32_t* cnt, int32_t* slot, void* ws, const Placement& pl, const DispatchArgs& d,
           cudaStream_t st) {
  const int nblk = T > 0 ? (T + BT - 1) / BT : 1;
  const size_t wbytes = (size_t)E * H * 2;
  const bool stage = E <= 16 && wbytes <= kMaxStagedW;  // (unstaged measured 10-50 % slower)
  const size_t smem = tail_smem_bytes(BT, E, pl.P) + (stage ? wbytes : 0);
  auto kern = stage ? gate_topk_kernel<TT, TE, true> : gate_topk_kernel<TT, TE, false>;
  if (int arc = smem_attr(reinterpret_cast<const void*>(kern), smem)) return arc;
  MSI_CUDA(launch_k(kern, dim3(nblk), dim3(kWarps * 32), smem, st, reinterpret_cast<const __nv_bfloat16*>(x),
                    reinterpret_cast<const __nv_bfloat16*>(wg), T, H, E, K, BT, idx, w, cnt, slot,
                    reinterpret_cast<int32_t*>(ws), pl, d));
  return check_launch("gate_topk_kernel");
}

// look-back words for the smallest BT (4) and the [T][E] fp32 logits scratch
// of the split path after them, 256-B aligned
size_t split_logits_offset(int T, int P) {
  const size_t nblk = ((size_t)T + 3) / 4 + 1;
  return (kLbOffset + nblk * (size_t)P * sizeof(uint64_t) + 255) & ~size_t(255);
}

template <int TT>
int launch_split(const void* x, const void* wg, int T, int H, int E, int K, int BTL, int EB, int32_t* idx,
                 float* w, int32_t* cnt, int32_t* slot, void* ws, const Placement& pl, const DispatchArgs& d,
                 cudaStream_t st) {
  constexpr int TE = 8;
  MSI_REQUIRE(BTL % TT == 0 && EB % TE == 0 && E % EB == 0, "gate_topk: bad split tile %dx%d", BTL, EB);
  float* logits = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + split_logits_offset(T, pl.P));
  const dim3 grid((T + BTL - 1) / BTL, E / EB);
  MSI_CUDA(launch_k(gate_logits_kernel<TT, TE>, grid, dim3(kWarps * 32), 0, st,
                    reinterpret_cast<const __nv_bfloat16*>(x), reinterpret_cast<const __nv_bfloat16*>(wg), T, H, E,
                    BTL, EB, logits, pl.pfw));
  constexpr int BT = 32;
  const size_t smem = tail_smem_bytes(BT, E, pl.P);
  if (int arc = smem_attr(reinterpret_cast<const void*>(route_kernel<1>), smem)) return arc;
  MSI_CUDA(launch_k(route_kernel<1>, dim3((T + BT - 1) / BT), dim3(kWarps * 32), smem, st,
                    reinterpret_cast<const __nv_bfloat16*>(x), (const float*)logits, T, E, K, BT, idx, w, cnt, slot,
                    reinterpret_cast<int32_t*>(ws), pl, d, (const __nv_bfloat16*)nullptr, (const float*)nullptr, H, 1));
  return check_launch("gate_logits_kernel + route_kernel");
}

// Tensor-core router for fine-grained MoE (E % 256 == 0, E <= 512): fp32
// logits on tcgen05 (dense_logits_f32, ~15 us for 4096 x 7168 x 256), then
// route_kernel recomputes only the candidate experts of every token in the
// pinned order (exactify) -- routing stays bit-exact with the oracle.
constexpr int kTcMaxSplit = 16;
size_t tc_norm_offset(int T, int P, int E) {
  return split_logits_offset(T, P) + (((size_t)kTcMaxSplit * T * E * sizeof(float) + 255) & ~size_t(255));
}

// split-K factor of the logits GEMM: enough units for the SMs (the N = E
// dimension is one or two 256-wide tiles), dividing H / 64
int tc_ksplit(int T, int E, int H) {
  const int units = ((T + 255) / 256) * (E / 256);  // CTA-pair tiles
  const int kb = H / 64;
  int best = 1;
  for (int sp = 1; sp <= kTcMaxSplit; ++sp)
    if (kb % sp == 0 && units * sp <= num_sms() / 2) best = sp;
  return best;
}

int route_tc(const void* x, const void* wg, int T, int H, int E, int K, int32_t* idx, float* w, int32_t* cnt,
             int32_t* slot, void* ws, const Placement& pl, const DispatchArgs& d, cudaStream_t st) {
  char* wsb = reinterpret_cast<char*>(ws);
  float* logits = reinterpret_cast<float*>(wsb + split_logits_offset(T, pl.P));
  float* wnorm = reinterpret_cast<float*>(wsb + tc_norm_offset(T, pl.P, E));
  MSI_CUDA(launch_k(wg_norm_kernel, dim3(E), dim3(256), 0, st, reinterpret_cast<const __nv_bfloat16*>(wg), H, wnorm));
  if (int rc = check_launch("wg_norm_kernel")) return rc;
  // ws word 4: the GEMM's tile counter (0 at rest; the launch's last fetch resets it)
  const int ksplit = tc_ksplit(T, E, H);
  if (int rc = dense_logits_f32(x, T, wg, E, H, logits, reinterpret_cast<uint32_t*>(wsb) + 4, st, ksplit)) return rc;
  // tokens per CTA: 4 up to T = 1024, 8 up to 2048, 16 above (the candidate
  // recompute is L2-latency-bound per warp, so more CTAs win until they
  // exceed 2 per SM; scripts/ab_router_lib.py, profiles/r02_ab_router_*.jsonl)
  int BT = T <= 1024 ? 4 : (T <= 2048 ? 8 : 16);
  if (const char* ov = getenv("MSI_ROUTER_TC_BT")) BT = std::max(4, std::min(32, atoi(ov)));
  const size_t smem = tail_smem_bytes(BT, E, pl.P) + (((size_t)BT * E + 7) & ~size_t(7)) * 2 + 32 * sizeof(int);
  auto kern = E <= 256 ? route_kernel<8> : route_kernel<16>;
  if (int arc = smem_attr(reinterpret_cast<const void*>(kern), smem)) return arc;
  MSI_CUDA(launch_k(kern, dim3((T + BT - 1) / BT), dim3(kWarps * 32), smem, st,
                    reinterpret_cast<const __nv_bfloat16*>(x), (const float*)logits, T, E, K, BT, idx, w, cnt, slot,
                    reinterpret_cast<int32_t*>(ws), pl, d, reinterpret_cast<const __nv_bfloat16*>(wg),
                    (const float*)wnorm, H, ksplit));
  return check_launch("route_kernel (tensor-core logits)");
}

// MSI_ROUTER_TC=1 forces the tensor-core path (when the shape allows), =0
// disables it; default: on for E % 256 == 0 from T >= 64 (DS-V3 shape, back-to-
// back medians vs the pinned-order CUDA-core path: T = 64 51 vs 56 us, 256 56
// vs 83, 1024 69 vs 136, 2048 91 vs 263, 4096 147 vs 454)
bool tc_enabled(int E, int T, int H) {
  if (E % 256 || E > 512 || H % 64) return false;
  const char* ov = getenv("MSI_ROUTER_TC");
  if (ov) return ov[0] == '1';
  return T >= 64;
}

// Split-path tiles: TT tokens per warp tile (TE = 8 experts), BTL tokens x EB
// experts per CTA.  MSI_ROUTER_SPLIT=TTxBTLxEB forces the split path with that
// tile (any T), =0 forces the fused kernel.
int route_split(const void* x, const void* wg, int T, int H, int E, int K, int32_t* idx, float* w, int32_t* cnt,
                int32_t* slot, void* ws, const Placement& pl, const DispatchArgs& d, cudaStream_t st) {
  // measured best at small T (scripts/sweep_router_split.py, T = 128: 2x4x32)
  int tt = 2, btl = 4, eb = 32;
  if (const char* ov = getenv("MSI_ROUTER_SPLIT")) {
    int a = 0, b = 0, c = 0;
    if (sscanf(ov, "%dx%dx%d", &a, &b, &c) == 3) { tt = a; btl = b; eb = c; }
  }
  if (E % eb) eb = 8;
  if (tt == 4) return launch_split<4>(x, wg, T, H, E, K, btl, eb, idx, w, cnt, slot, ws, pl, d, st);
  if (tt == 2) return launch_split<2>(x, wg, T, H, E, K, btl, eb, idx, w, cnt, slot, ws, pl, d, st);
  return launch_split<1>(x, wg, T, H, E, K, btl, eb, idx, w, cnt, slot, ws, pl, d, st);
}

// The split path wins only at small T (T = 128: 92 -> 71 us); from T ~ 512 on
// the fused kernel's W_g reuse across its 16-32 tokens is worth more than the
// split grid's occupancy (profiles/r01_router_split_sweep.jsonl).
bool split_enabled(int E, int T) {
  const char* ov = getenv("MSI_ROUTER_SPLIT");
  if (ov) return ov[0] != '0';
  return E >= 64 && E % 8 == 0 && T <= 256;
}

}  // namespace

int gate_topk(const void* x, const void* wg, int T, int H, int E, int K, int32_t* idx, float* w,
              int32_t* cnt, int32_t* slot, void* ws, cudaStream_t st, const int32_t* rep, int R, int P, int sender,
              int32_t* pidx, const DispatchArgs* dp) {
  MSI_REQUIRE(T >= 0 && H > 0 && H % 256 == 0, "gate_topk: H must be a positive multiple of 256 (got %d)", H);
  MSI_REQUIRE(E >= 1 && E <= 1024 && K >= 1 && K <= E && K <= 32, "gate_topk: need 1 <= K <= min(E, 32), E <= 1024");
  // an empty micro-batch (T = 0) may pass null token / output buffers
  MSI_REQUIRE((x || T == 0) && wg && (T == 0 || (idx && w && slot)) && cnt && ws, "gate_topk: null pointer");
  MSI_REQUIRE(!rep || (R >= 1 && P >= E && P <= 4096 && pidx && sender >= 0),
              "gate_topk: replica table needs R >= 1, E <= P <= 4096, pidx and sender >= 0");
  const char* pf = getenv("MSI_ROUTER_PFW");
  const Placement pl{rep, R, rep ? P : E, sender, rep ? pidx : idx, (pf && pf[0] == '1') ? 1 : 0};
  DispatchArgs d{};
  if (dp) d = *dp;
  if (T == 0 && !d.on) {
    MSI_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * pl.P, st));
    return 0;
  }
  if (T == 0)  // empty micro-batch with dispatch: one CTA still runs the protocol (zero counts, release)
    return launch<1, 1>(x, wg, 0, H, E, K, 8, idx, w, cnt, slot, ws, pl, d, st);
  // Tile shapes: TE experts x TT tokens per warp; BT tokens per CTA.  Small E
  // is HBM-bound (want many CTAs); large E is FMA-bound (want token reuse).
  // MSI_ROUTER_TILE=TTxTExBT overrides the choice (tuning experiments).
  if (const char* ov = getenv("MSI_ROUTER_TILE")) {
    int tt = 0, te = 0, bt = 0;
    if (sscanf(ov, "%dx%dx%d", &tt, &te, &bt) == 3 && bt >= 4 && bt >= tt && bt <= 32 && bt % tt == 0 && E % te == 0) {
#define MSI_RT(A, B) if (tt == A && te == B) return launch<A, B>(x, wg, T, H, E, K, bt, idx, w, cnt, slot, ws, pl, d, st);
      MSI_RT(1, 8) MSI_RT(2, 8) MSI_RT(4, 8) MSI_RT(8, 8) MSI_RT(1, 16) MSI_RT(2, 16) MSI_RT(4, 16) MSI_RT(8, 4)
      MSI_RT(4, 4) MSI_RT(2, 4)
#undef MSI_RT
    }
  }
  // fine-grained MoE at small T: logits on their own 2-D grid, then top-K /
  // placement (route_split)
  if (tc_enabled(E, T, H)) return route_tc(x, wg, T, H, E, K, idx, w, cnt, slot, ws, pl, d, st);
  if (split_enabled(E, T) && E >= 64 && E % 8 == 0) return route_split(x, wg, T, H, E, K, idx, w, cnt, slot, ws, pl, d, st);
  // One CTA per SM fits (255 registers): BT = the smallest multiple of 4 that
  // covers T in one wave of num_sms() CTAs (<= 32), so no second partial wave
  // (T = 4096: BT 16 -> 28, 256 -> 147 CTAs) and W_g is re-read by as few
  // CTAs as possible
  if (E % 16 == 0 && E > 16) {
    int bt = 4 * ((T + 4 * num_sms() - 1) / (4 * num_sms()));
    bt = bt < 4 ? 4 : (bt > 32 ? 32 : bt);
    return launch<4, 16>(x, wg, T, H, E, K, bt, idx, w, cnt, slot, ws, pl, d, st);
  }
  // E = 8 / 16: W_g staged once per CTA (TMA bulk copy) and amortised over 32
  // tokens (4 per warp); x is the only HBM stream
  // (BT shrinks for small T so that ~100+ CTAs stream x: measured with
  //  scripts/sweep_router_tiles.py -- DBRX T=1024: 50 -> 32 us at BT = 8)
  const int bt = T >= 96 * 32 ? 32 : (T >= 96 * 16 ? 16 : 8);
  if (E % 16 == 0) {
    if (bt == 32) return launch<4, 16>(x, wg, T, H, E, K, 32, idx, w, cnt, slot, ws, pl, d, st);
    if (bt == 16) return launch<2, 16>(x, wg, T, H, E, K, 16, idx, w, cnt, slot, ws, pl, d, st);
    return launch<1, 16>(x, wg, T, H, E, K, 8, idx, w, cnt, slot, ws, pl, d, st);
  }
  if (E % 8 == 0) {
    if (bt == 32) return launch<4, 8>(x, wg, T, H, E, K, 32, idx, w, cnt, slot, ws, pl, d, st);
    if (bt == 16) return launch<2, 8>(x, wg, T, H, E, K, 16, idx, w, cnt, slot, ws, pl, d, st);
    return launch<1, 8>(x, wg, T, H, E, K, 8, idx, w, cnt, slot, ws, pl, d, st);
  }
  if (E % 4 == 0) return launch<1, 4>(x, wg, T, H, E, K, 8, idx, w, cnt, slot, ws, pl, d, st);
  if (E % 2 == 0) return launch<1, 2>(x, wg, T, H, E, K, 8, idx, w, cnt, slot, ws, pl, d, st);
  return launch<1, 1>(x, wg, T, H, E, K, 8, idx, w, cnt, slot, ws, pl, d, st);
}

size_t gate_topk_workspace(int T, int E) {
  // look-back words for the smallest BT (4); split path (E >= 64): + [T][E]
  // fp32 logits (E here is the physical slot count P >= logical E)
  const size_t lb = split_logits_offset(T, E);
  // + the tensor-core path's per-expert norms after the logits
  return E >= 64 ? tc_norm_offset(T, E, E) + (size_t)E * sizeof(float) : lb;
}

}  // namespace msi

extern "C" size_t msi_gate_topk_workspace(int T, int E) { return msi::gate_topk_workspace(T, E); }

extern "C" int msi_gate_topk(const void* x, const void* wg, int T, int H, int E, int K,
                             int32_t* idx, float* w, int32_t* cnt, int32_t* slot, void* workspace,
                             void* stream) {
  return msi::gate_topk(x, wg, T, H, E, K, idx, w, cnt, slot, workspace,
                        reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int msi_gate_topk_placed(const void* x, const void* wg, int T, int H, int E, int K,
                                    const int32_t* rep, int R, int P, int sender, int32_t* idx,
                                    int32_t* pidx, float* w, int32_t* cnt, int32_t* slot,
                                    void* workspace, void* stream) {
  return msi::gate_topk(x, wg, T, H, E, K, idx, w, cnt, slot, workspace,
                        reinterpret_cast<cudaStream_t>(stream), rep, R, P, sender, pidx);
}
