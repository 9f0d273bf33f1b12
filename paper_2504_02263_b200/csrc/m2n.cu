// m2n.cu -- M2N dispatch / N2M combine over NVLink peer memory, the symmetric
// heap and its IPC registration, and the expert-step driver.
//
// The paper's M2N library moves tokens with CPU-driven
// RDMA: the sender waits on a CUDA event, blocks its stream with a driver op,
// has a CPU "core sender" post RDMA writes-with-immediate and poll the CQ,
// then unblocks the stream; the receiver polls its CQ, flushes
// with GDRCopy and unblocks.  On one NVSwitch box none of
// that machinery is needed: every GPU maps every peer's receive buffers once
// (CUDA IPC, the "pre-registered tensor"), SMs store rows straight into peer
// HBM with 16 B vector stores, and readiness is a monotone epoch counter
// bumped with red.release.sys and polled with ld.acquire.sys -- no host in the
// loop, no per-step setup.
//
// Heap layout of one rank (offsets identical on every rank of the same role):
//   ctrl   : per-slot counters, one 128 B line each
//            arrive[slot]  (expert role)    dispatch arrivals, +1 per sender
//            comb[slot]    (attention role) combine arrivals, +1 per expert GPU
//            dticket[slot], fticket[slot]   last-CTA tickets (local)
//            ause[slot], euse[slot]         uses of each slot so far (attention /
//                                           expert side): epoch 0 in the ABI means
//                                           "next use", read on the device, so a
//                                           whole step can be captured in a CUDA graph
//            status[2]                      device error word + abort flag
//            stats[2] u64                   rows through the expert FFN, FFN calls
//            cntab[slot][n_a][E] u64        (epoch << 32 | count), all-gathered
//   recv   : (expert role)    [slot][E_l][n_a][max_tokens][H] bf16 received rows:
//            one region per (local expert, sender), so a sender places its
//            rows from its own counts alone (no count exchange before the
//            payload); the expert GEMM loads a tile's rows as runs of these
//            regions (TMA boxes at any row offset), and GEMM2 writes each Y
//            row over its X -- the attention GPU's combine pulls it from
//            there (it knows the row from its own routing), so there is no
//            per-row metadata and no combine buffer
//   hbuf   : (expert role, separate allocation) [cap][H'] SwiGLU activations,
//            per-expert segments 128-row aligned in virtual (sender-major)
//            row order; cap = n_a * max_tokens * min(K, E_l) + E_l * 127.
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "gemm.h"
#include "route.h"
#include "tp.h"

namespace msi {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s launch: %s", what, cudaGetErrorString(e));
    return (int)e;
  }
  return 0;
}

int smem_attr(const void* fn, size_t bytes) {
  if (bytes <= 48 * 1024) return 0;
  struct Entry { const void* fn; int dev; size_t bytes; };
  static std::mutex mu;
  static std::vector<Entry> done;
  int dev = 0;
  MSI_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  for (Entry& e : done)
    if (e.fn == fn && e.dev == dev) {
      if (e.bytes >= bytes) return 0;
      MSI_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
      e.bytes = bytes;
      return 0;
    }
  MSI_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  done.push_back({fn, dev, bytes});
  return 0;
}

// MSI_REGION_RUNS=1: GEMM1 loads several senders' regions as box runs
// instead of gathering them first (A/B runs; measured slower).
bool region_runs_forced() {
  const char* e = getenv("MSI_REGION_RUNS");
  return e && e[0] == '1';
}

bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MSI_PDL");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

namespace {

constexpr int CTR_STRIDE = 32;  // u32 per counter line (128 B)
constexpr size_t ALIGN = 4096;

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Expert tensor parallelism: tp GPUs form an expert node sharing its experts.
inline int plan_tp(const msi_plan& p) { return p.tp_e > 1 ? p.tp_e : 1; }
inline int plan_nodes(const msi_plan& p) { return p.n_e / plan_tp(p); }
inline int plan_el(const msi_plan& p) { return p.experts / plan_nodes(p); }
inline int plan_tpa(const msi_plan& p) { return p.tp_a > 1 ? p.tp_a : 1; }

struct Layout {
  size_t arrive, comb, dticket, fticket, ause, euse, status, stats, trace, cntab, ctrl_bytes;
  size_t tpready, tprs, tpuse, tpticket;  // attention TP counters (per slot lines)
  size_t tpx, tpx_slot, tprsb, tprsb_slot;  // attention TP: shard [cap][H], partials [tp][cap][H] per slot
  size_t recv, recv_slot;
  size_t total;
  int64_t cap;       // hbuf rows (compact, 128-aligned segments)
  int64_t recv_rows;  // recv rows per slot: E_l * n_a * max_tokens
};

Layout make_layout(const msi_plan& p, bool attn, bool expert) {
  Layout L{};
  const size_t line = CTR_STRIDE * 4;
  size_t off = 0;
  L.arrive = off; off += p.slots * line;
  L.comb = off; off += p.slots * line;
  L.dticket = off; off += p.slots * line;
  L.fticket = off; off += p.slots * line;
  L.ause = off; off += p.slots * line;
  L.euse = off; off += p.slots * line;
  L.status = off; off += line;
  L.stats = off; off += line;
  L.trace = off; off += 2 * line;  // 32 x u64 %globaltimer stamps
  L.cntab = off; off += (size_t)p.slots * p.n_a * p.experts * 8;
  L.tpready = off; off += p.slots * line;
  L.tprs = off; off += p.slots * line;
  L.tpuse = off; off += p.slots * line;
  L.tpticket = off; off += p.slots * line;
  L.ctrl_bytes = align_up(off, ALIGN);
  off = L.ctrl_bytes;
  if (attn && plan_tpa(p) > 1) {  // before the expert buffers: same offsets on every attention GPU
    L.tpx_slot = (size_t)p.max_tokens * p.hidden * 2;
    L.tpx = off; off += align_up(L.tpx_slot * p.slots, ALIGN);
    L.tprsb_slot = (size_t)plan_tpa(p) * L.tpx_slot;
    L.tprsb = off; off += align_up(L.tprsb_slot * p.slots, ALIGN);
  }
  const int E_l = plan_el(p);  // experts per expert node (tp_e GPUs share them)
  const int per_tok = p.topk < E_l ? p.topk : E_l;
  int64_t cap = (int64_t)p.n_a * p.max_tokens * per_tok + (int64_t)E_l * (MSI_ROW_ALIGN - 1);
  L.cap = (cap + 127) / 128 * 128;
  L.recv_rows = (int64_t)E_l * p.n_a * p.max_tokens;
  L.recv_slot = (size_t)L.recv_rows * p.hidden * 2;
  L.recv = off;
  if (expert) off += align_up(L.recv_slot * p.slots, ALIGN);
  L.total = off;
  return L;
}

// Everything a device kernel needs, by value (kernel parameter space).
struct DevCtx {
  int n_a, n_e, n_world, E, K, H, Hp, E_l, slots, max_tokens;
  int my_a, my_e;
  int tp, nodes, my_node, my_tp;  // expert TP: node = tp GPUs; this GPU's node and rank in it
  long long cap;        // hbuf rows
  long long recv_rows;  // recv rows per slot (E_l * n_a * max_tokens regions)
  uint64_t timeout_ns;
  uint64_t* ecntab_of[MSI_MAX_RANKS];  // count table per expert index q
  uint32_t* arrive_of[MSI_MAX_RANKS];  // per expert index q
  char* recv_of[MSI_MAX_RANKS];        // per expert index q
  uint32_t* comb_of[MSI_MAX_RANKS];    // per attention index s
  uint64_t* my_cntab;
  uint32_t *my_arrive, *my_comb, *my_dticket, *my_fticket, *my_ause, *my_euse;
  int32_t* my_status;
  unsigned long long* trace;  // null = tracing off
  // attention TP (plan.tp_a > 1): this GPU's node peers j = 0..tp_a-1
  int tp_a, my_ta;
  char* tpx_of[MSI_MAX_RANKS];        // peer j's shard buffers (slot 0)
  char* tprsb_of[MSI_MAX_RANKS];      // peer j's partial buffers (slot 0)
  uint32_t* tpready_of[MSI_MAX_RANKS];
  uint32_t* tprs_of[MSI_MAX_RANKS];
  uint32_t *my_tpready, *my_tprs, *my_tpuse, *my_tpticket;
};

}  // namespace
}  // namespace msi

struct msi_ctx {
  msi_plan plan;
  int rank;
  bool attn, expert;
  int my_a, my_e;
  char* heap = nullptr;
  char* hbuf = nullptr;       // expert role: SwiGLU activations [cap][H']
  char* xcomp = nullptr;      // expert role with n_a > 1: gathered rows [cap][H] (GEMM1's A)
  void* workspace = nullptr;  // router workspace for the runtime (zeroed)
  size_t ws_bytes = 0;
  size_t heap_bytes = 0;
  char* peer[MSI_MAX_RANKS] = {nullptr};
  bool opened[MSI_MAX_RANKS] = {false};
  bool finalized = false;
  uint64_t timeout_ns = 20ull * 1000 * 1000 * 1000;
  msi::Layout my_layout;
  msi::DevCtx dev;
};

namespace msi {
namespace {

bool role_attn(const msi_plan& p, int r) {
  for (int i = 0; i < p.n_a; ++i) if (p.attn_ranks[i] == r) return true;
  return false;
}
bool role_expert(const msi_plan& p, int r) {
  for (int i = 0; i < p.n_e; ++i) if (p.expert_ranks[i] == r) return true;
  return false;
}

int validate(const msi_plan& p) {
  MSI_REQUIRE(p.world >= 1 && p.world <= MSI_MAX_RANKS, "plan: world must be in [1, %d]", MSI_MAX_RANKS);
  MSI_REQUIRE(p.n_a >= 1 && p.n_a <= p.world && p.n_e >= 1 && p.n_e <= p.world, "plan: bad n_a/n_e");
  MSI_REQUIRE(p.tp_e >= 0 && p.tp_e <= p.n_e && p.n_e % plan_tp(p) == 0, "plan: tp_e must divide n_e");
  MSI_REQUIRE(p.tp_a >= 0 && p.tp_a <= MSI_MAX_RANKS && p.n_a % plan_tpa(p) == 0, "plan: tp_a must divide n_a");
  MSI_REQUIRE(p.experts >= 1 && p.experts % plan_nodes(p) == 0, "plan: experts must divide over the expert nodes");
  MSI_REQUIRE(plan_el(p) <= MSI_MAX_LOCAL_EXPERTS, "plan: at most %d experts per GPU", MSI_MAX_LOCAL_EXPERTS);
  MSI_REQUIRE(p.inter % (128 * plan_tp(p)) == 0, "plan: inter must split into tp_e multiples of 128");
  MSI_REQUIRE(p.topk * plan_tp(p) <= 32, "plan: topk * tp_e <= 32");
  MSI_REQUIRE(p.topk >= 1 && p.topk <= p.experts && p.topk <= 32, "plan: bad topk");
  MSI_REQUIRE(p.hidden % 256 == 0 && p.inter % 128 == 0, "plan: hidden %% 256 and inter %% 128 required");
  MSI_REQUIRE(p.max_tokens >= 1 && p.slots >= 1 && p.slots <= 16, "plan: bad max_tokens/slots");
  for (int i = 0; i < p.n_a; ++i) MSI_REQUIRE(p.attn_ranks[i] >= 0 && p.attn_ranks[i] < p.world, "plan: attn rank out of range");
  for (int i = 0; i < p.n_e; ++i) MSI_REQUIRE(p.expert_ranks[i] >= 0 && p.expert_ranks[i] < p.world, "plan: expert rank out of range");
  return 0;
}

// ------------------------------------------------------------ dispatch ----
constexpr int kDispThreads = 512;

// Stand-alone M2N dispatch (msi_dispatch: router outputs given).  Row (t, k)
// goes to region (e_l, s) of its expert GPU at its slot -- this sender's own
// counts place it, so no other sender is waited for; the last CTA publishes
// the counts (tagged with the epoch) to every expert GPU and releases their
// arrival counters.  The fused router + dispatch (msi_route_dispatch,
// router.cu) does the same from inside the router.
__global__ void __launch_bounds__(kDispThreads)
dispatch_kernel(const DevCtx c, const __nv_bfloat16* __restrict__ x, const int32_t* __restrict__ cnt,
                const int32_t* __restrict__ idx, const int32_t* __restrict__ slot, int T, int mb,
                uint32_t epoch) {
  __shared__ uint32_t s_epoch;
  __shared__ int s_last;
  const int tid = threadIdx.x;
  pdl_trigger();
  pdl_wait();
  if (tid == 0) s_epoch = resolve_epoch(epoch, c.my_ause + mb * CTR_STRIDE, 1u, c.my_status);
  __syncthreads();
  epoch = s_epoch;
  if (epoch == 0) return;  // host/device epoch mismatch: status set, nothing sent
  const int s = c.my_a;
  if (blockIdx.x == 0 && tid == 0) trace_stamp(c.trace, 0);
  const int lane = tid & 31;
  const int gwarp = blockIdx.x * (blockDim.x >> 5) + (tid >> 5);
  const int nwarps = gridDim.x * (blockDim.x >> 5);
  const size_t row_bytes = (size_t)c.H * 2;
  // a warp moves one part of one token row (x read once, written K * tp
  // times with 16 B stores, 8 x 512 B in flight per warp)
  const int nchunk = c.H >> 8;  // 512 B warp-chunks per row
  int parts = T > 0 ? (nwarps + T - 1) / T : 1;
  parts = parts < 1 ? 1 : (parts > nchunk ? nchunk : parts);
  const int per_part = (nchunk + parts - 1) / parts;
  for (int item = gwarp; item < T * parts; item += nwarps) {
    const int t = item / parts, part = item - t * parts;
    // lane j (< K * tp) resolves destination j: (t, k = j / tp) on GPU r = j % tp
    // of expert node e / E_l (every GPU of a node receives the row)
    char* my_dst = nullptr;
    const int ndst = c.K * c.tp;
    if (lane < ndst) {
      const int k = lane / c.tp, r = lane - (lane / c.tp) * c.tp;
      const int e = idx[(size_t)t * c.K + k];
      const int q = (e / c.E_l) * c.tp + r;
      const long long row = (long long)mb * c.recv_rows +
                            ((long long)(e % c.E_l) * c.n_a + s) * c.max_tokens + slot[(size_t)t * c.K + k];
      my_dst = c.recv_of[q] + (size_t)row * row_bytes;
    }
    const char* src = reinterpret_cast<const char*>(x + (size_t)t * c.H) + lane * 16;
    const int j_end = min(nchunk, (part + 1) * per_part);
    constexpr int U = 8;
    for (int j0 = part * per_part; j0 < j_end; j0 += U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (j0 + u < j_end) v[u] = ld_nc_v4(src + (size_t)(j0 + u) * 512);
      for (int k = 0; k < ndst; ++k) {
        char* d = reinterpret_cast<char*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(my_dst), k)) + lane * 16;
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (j0 + u < j_end) st_v4(d + (size_t)(j0 + u) * 512, v[u]);
      }
    }
  }

  // ---- the last CTA: counts to every expert GPU, then release -------------
  __syncthreads();
  if (tid == 0) {
    __threadfence_system();
    s_last = atomicAdd(c.my_dticket + mb * CTR_STRIDE, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  const size_t tab = (size_t)mb * c.n_a * c.E;
  for (int i = tid; i < c.n_e * c.E; i += blockDim.x) {
    const int q = i / c.E, e = i - q * c.E;
    st_relaxed_sys64(c.ecntab_of[q] + tab + (size_t)s * c.E + e, ((uint64_t)epoch << 32) | (uint32_t)cnt[e]);
  }
  __syncthreads();
  if (tid == 0) {
    c.my_dticket[mb * CTR_STRIDE] = 0;
    c.my_ause[mb * CTR_STRIDE] = epoch;  // every CTA has read the old value
    trace_stamp(c.trace, 2);
    fence_sys();
    for (int q = 0; q < c.n_e; ++q) red_release_sys_add(c.arrive_of[q] + mb * CTR_STRIDE, 1u);
  }
}

// ---------------------------------------------------------------- echo ----
// Identity expert (Y = X): waits for every sender's rows like the expert FFN
// and releases the attention GPUs the same way, without touching the rows --
// the combine then pulls X back from the receive regions.  dispatch + echo +
// combine is the pure M2N round trip (both legs' bytes over NVLink).
// Expert-side wait for a slot's rows (one thread): spins until every sender
// released the slot's epoch (device-resolved like msi_expert_ffn's), so the
// FFN kernels that follow start on data already in place and their timing is
// compute only.  On timeout it sets the abort flag the FFN kernels honour.
__global__ void expert_wait_kernel(const DevCtx c, int mb, uint32_t epoch) {
  pdl_trigger();
  pdl_wait();
  epoch = resolve_epoch(epoch, c.my_euse + mb * CTR_STRIDE, 1u, c.my_status);
  if (epoch == 0) return;  // the FFN kernels see the same mismatch and abort
  if (!wait_geq(c.my_arrive + mb * CTR_STRIDE, epoch * (uint32_t)c.n_a, c.timeout_ns, c.my_status))
    c.my_status[1] = 1;
}

__global__ void echo_kernel(const DevCtx c, int mb, uint32_t epoch) {
  pdl_trigger();
  pdl_wait();
  epoch = resolve_epoch(epoch, c.my_euse + mb * CTR_STRIDE, 1u, c.my_status);
  if (epoch == 0) return;
  trace_stamp(c.trace, 3);
  if (!wait_geq(c.my_arrive + mb * CTR_STRIDE, epoch * (uint32_t)c.n_a, c.timeout_ns, c.my_status)) return;
  trace_stamp(c.trace, 4);
  c.my_euse[mb * CTR_STRIDE] = epoch;
  trace_stamp(c.trace, 5);
  fence_sys();
  for (int s = 0; s < c.n_a; ++s) red_release_sys_add(c.comb_of[s] + mb * CTR_STRIDE, 1u);
}

// ------------------------------------------------------------- combine ----
// N2M combine as a pull: the attention GPU reads the K (x tp partial) expert
// output rows of each token straight from the expert GPUs' receive regions
// (NVLink peer loads; SM loads pull 750 GB/s one way against 700 for stores,
// scripts/peer_load_probe.cu) and reduces them on the fly, so the return leg
// and the weighted sum are one pass and no combine buffer is written.
// out[t] = bf16(resid[t] + sum_{k, r} w[t,k] * y[t,k,r]), fp32 fmaf in
// ascending (k, r) -- the oracle's order.
struct CombineSrc {
  const char* y[MSI_MAX_RANKS];  // per expert GPU q: rows of this micro-batch slot
  int E_l, tp, n_send, s;        // row of (t, k): ((p % E_l) * n_send + s) * cap_s + slot
  long long cap_s;
  const int32_t* dest;           // [T, K] physical slot (null: rows [T, K(, tp)] of y[0])
  const int32_t* slot;           // [T, K]
};

template <int KR>
__device__ __forceinline__ void combine_row8(const CombineSrc& src, const float* w, const uint16_t* resid, uint16_t* out,
                                             int t, int col8, int K, int H, uint4* gather) {
  uint4 y[KR];
  float wk[KR];
#pragma unroll
  for (int kr = 0; kr < KR; ++kr) {
    const int k = kr / src.tp, r = kr - k * src.tp;
    const char* row;
    if (src.dest) {
      const int p = src.dest[(size_t)t * K + k];
      const long long rr = ((long long)(p % src.E_l) * src.n_send + src.s) * src.cap_s + src.slot[(size_t)t * K + k];
      row = src.y[(p / src.E_l) * src.tp + r] + (size_t)rr * H * 2;
    } else {
      row = src.y[0] + ((size_t)t * KR + kr) * H * 2;
    }
    y[kr] = __ldcg(reinterpret_cast<const uint4*>(row + (size_t)col8 * 16));
    wk[kr] = w ? w[(size_t)t * K + k] : 0.0f;
  }
  if (gather) {  // msi_gather_y: the rows themselves, [T][K*tp][H]
#pragma unroll
    for (int kr = 0; kr < KR; ++kr) gather[((size_t)t * KR + kr) * (H / 8) + col8] = y[kr];
    return;
  }
  float acc[8];
  if (resid) {
    uint4 r = *reinterpret_cast<const uint4*>(resid + (size_t)t * H + col8 * 8);
    acc[0] = bf16lo(r.x); acc[1] = bf16hi(r.x); acc[2] = bf16lo(r.y); acc[3] = bf16hi(r.y);
    acc[4] = bf16lo(r.z); acc[5] = bf16hi(r.z); acc[6] = bf16lo(r.w); acc[7] = bf16hi(r.w);
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
  }
#pragma unroll
  for (int kr = 0; kr < KR; ++kr) {
    acc[0] = __fmaf_rn(wk[kr], bf16lo(y[kr].x), acc[0]); acc[1] = __fmaf_rn(wk[kr], bf16hi(y[kr].x), acc[1]);
    acc[2] = __fmaf_rn(wk[kr], bf16lo(y[kr].y), acc[2]); acc[3] = __fmaf_rn(wk[kr], bf16hi(y[kr].y), acc[3]);
    acc[4] = __fmaf_rn(wk[kr], bf16lo(y[kr].z), acc[4]); acc[5] = __fmaf_rn(wk[kr], bf16hi(y[kr].z), acc[5]);
    acc[6] = __fmaf_rn(wk[kr], bf16lo(y[kr].w), acc[6]); acc[7] = __fmaf_rn(wk[kr], bf16hi(y[kr].w), acc[7]);
  }
  uint4 o = make_uint4(pack_bf16x2(acc[0], acc[1]), pack_bf16x2(acc[2], acc[3]),
                       pack_bf16x2(acc[4], acc[5]), pack_bf16x2(acc[6], acc[7]));
  *reinterpret_cast<uint4*>(out + (size_t)t * H + col8 * 8) = o;
}

template <int KR>
__global__ void __launch_bounds__(256)
combine_kernel(const CombineSrc src, const float* __restrict__ w, const uint16_t* __restrict__ resid,
               uint16_t* __restrict__ out, uint4* __restrict__ gather, int T, int K, int H, const uint32_t* wait_ctr,
               uint32_t epoch, uint32_t mul, const uint32_t* epoch_src, uint64_t timeout_ns, int32_t* status,
               unsigned long long* trace) {
  __shared__ int s_ok;
  const bool t0 = blockIdx.x == 0 && threadIdx.x == 0;
  pdl_trigger();
  pdl_wait();
  if (wait_ctr) {
    epoch = resolve_epoch(epoch, epoch_src, 0u, status);  // set by this slot's dispatch
    if (epoch == 0) return;
    if (t0) trace_stamp(trace, 6);
    if (threadIdx.x == 0) s_ok = wait_geq(wait_ctr, epoch * mul, timeout_ns, status);
    __syncthreads();
    if (!s_ok) return;
    if (t0) trace_stamp(trace, 7);
  }
  const int per_row = H / 8;
  const size_t n = (size_t)T * per_row;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    combine_row8<KR>(src, w, resid, out, (int)(i / per_row), (int)(i % per_row), K, H, gather);
  if (t0) trace_stamp(trace, 8);
}

template <int KR>
cudaError_t launch_combine_kr(const CombineSrc& src, const float* w, const void* resid, void* out, void* gather, int T,
                              int K, int H, const uint32_t* wait_ctr, uint32_t epoch, uint32_t mul,
                              const uint32_t* epoch_src, uint64_t timeout_ns, int32_t* status,
                              unsigned long long* trace, cudaStream_t st) {
  const size_t n = (size_t)T * H / 8;
  // 6 resident CTAs per SM (the 40-register occupancy limit): 36.2 vs 39.5 us
  // at 4 for the N = 1 bench step (profiles/r02_ab_combine.txt); MSI_COMBINE_CTAS
  static const int mult = [] {
    const char* v = getenv("MSI_COMBINE_CTAS");
    const int m = v ? atoi(v) : 6;
    return m >= 1 && m <= 8 ? m : 6;
  }();
  int grid = (int)((n + 255) / 256);
  grid = grid < 1 ? 1 : (grid > mult * num_sms() ? mult * num_sms() : grid);
  return launch_k(combine_kernel<KR>, dim3(grid), dim3(256), 0, st, src, w, reinterpret_cast<const uint16_t*>(resid),
                  reinterpret_cast<uint16_t*>(out), reinterpret_cast<uint4*>(gather), T, K, H, wait_ctr, epoch, mul,
                  epoch_src, timeout_ns, status, trace);
}

// K * tp rows per token; every supported count gets its own unrolled kernel
int launch_combine(const CombineSrc& src, const float* w, const void* resid, void* out, void* gather, int T, int K,
                   int H, const uint32_t* wait_ctr, uint32_t epoch, uint32_t mul, const uint32_t* epoch_src,
                   uint64_t timeout_ns, int32_t* status, unsigned long long* trace, cudaStream_t st) {
  cudaError_t e;
  switch (K * src.tp) {
#define MSI_KR(N) case N: e = launch_combine_kr<N>(src, w, resid, out, gather, T, K, H, wait_ctr, epoch, mul, epoch_src, \
                                                  timeout_ns, status, trace, st); break;
    MSI_KR(1) MSI_KR(2) MSI_KR(3) MSI_KR(4) MSI_KR(5) MSI_KR(6) MSI_KR(7) MSI_KR(8) MSI_KR(12) MSI_KR(16)
    MSI_KR(24) MSI_KR(32)
#undef MSI_KR
    default:
      set_error("combine: K * tp_e = %d rows per token unsupported", K * src.tp);
      return MSI_EINVAL;
  }
  if (e != cudaSuccess) { set_error("combine launch: %s", cudaGetErrorString(e)); return (int)e; }
  return check_launch("combine_kernel");
}

}  // namespace
}  // namespace msi

using namespace msi;

// =============================================================== C ABI ====
extern "C" int msi_version(void) { return 1; }
extern "C" const char* msi_last_error(void) { return msi::g_err; }

extern "C" int msi_check_device(void) {
  int dev = 0, major = 0, minor = 0;
  MSI_CUDA(cudaGetDevice(&dev));
  MSI_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  MSI_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev));
  if (major != 10 || minor != 0) {
    set_error("libmsinfer is built for sm_100a (B200); device is sm_%d%d", major, minor);
    return MSI_EARCH;
  }
  return 0;
}

extern "C" int msi_ctx_create(const msi_plan* plan, int rank, msi_ctx** out) {
  if (!plan || !out) { set_error("msi_ctx_create: null argument"); return MSI_EINVAL; }
  int rc = validate(*plan);
  if (rc) return rc;
  if (rank < 0 || rank >= plan->world) { set_error("msi_ctx_create: rank out of range"); return MSI_EINVAL; }
  rc = msi_check_device();
  if (rc) return rc;
  msi_ctx* c = new msi_ctx();
  c->plan = *plan;
  c->rank = rank;
  c->attn = role_attn(*plan, rank);
  c->expert = role_expert(*plan, rank);
  c->my_a = c->my_e = -1;
  for (int i = 0; i < plan->n_a; ++i) if (plan->attn_ranks[i] == rank) c->my_a = i;
  for (int i = 0; i < plan->n_e; ++i) if (plan->expert_ranks[i] == rank) c->my_e = i;
  c->my_layout = make_layout(*plan, c->attn, c->expert);
  c->heap_bytes = c->my_layout.total;
  auto fail = [&](const char* what, cudaError_t e) {
    set_error("msi_ctx_create: %s: %s", what, cudaGetErrorString(e));
    if (c->heap) cudaFree(c->heap);
    if (c->hbuf) cudaFree(c->hbuf);
    if (c->xcomp) cudaFree(c->xcomp);
    if (c->workspace) cudaFree(c->workspace);
    delete c;
    return (int)e;
  };
  cudaError_t e = cudaMalloc(&c->heap, c->heap_bytes);
  if (e != cudaSuccess) return fail("heap cudaMalloc", e);
  if ((e = cudaMemset(c->heap, 0, c->my_layout.ctrl_bytes)) != cudaSuccess) return fail("heap memset", e);
  if (c->expert) {
    e = cudaMalloc(&c->hbuf, (size_t)c->my_layout.cap * plan->inter * 2);
    if (e != cudaSuccess) return fail("hbuf cudaMalloc", e);
    if (plan->n_a > 1) {
      e = cudaMalloc(&c->xcomp, (size_t)c->my_layout.cap * plan->hidden * 2);
      if (e != cudaSuccess) return fail("xcomp cudaMalloc", e);
    }
  }
  c->ws_bytes = msi_gate_topk_workspace(plan->max_tokens, plan->experts);
  if ((e = cudaMalloc(&c->workspace, c->ws_bytes)) != cudaSuccess) return fail("workspace cudaMalloc", e);
  if ((e = cudaMemset(c->workspace, 0, c->ws_bytes)) != cudaSuccess) return fail("workspace memset", e);
  c->peer[rank] = c->heap;
  c->opened[rank] = true;
  *out = c;
  return 0;
}

extern "C" int msi_ctx_destroy(msi_ctx* c) {
  if (!c) return 0;
  cudaDeviceSynchronize();
  for (int r = 0; r < c->plan.world; ++r)
    if (r != c->rank && c->opened[r] && c->peer[r]) cudaIpcCloseMemHandle(c->peer[r]);
  if (c->heap) cudaFree(c->heap);
  if (c->hbuf) cudaFree(c->hbuf);
  if (c->xcomp) cudaFree(c->xcomp);
  if (c->workspace) cudaFree(c->workspace);
  delete c;
  return 0;
}

extern "C" int msi_ctx_export(msi_ctx* c, msi_ipc_handle* out) {
  static_assert(sizeof(cudaIpcMemHandle_t) == MSI_IPC_HANDLE_BYTES, "ipc handle size");
  if (!c || !out) { set_error("msi_ctx_export: null argument"); return MSI_EINVAL; }
  cudaIpcMemHandle_t h;
  MSI_CUDA(cudaIpcGetMemHandle(&h, c->heap));
  memcpy(out->bytes, &h, sizeof(h));
  return 0;
}

extern "C" int msi_ctx_import(msi_ctx* c, int peer, const msi_ipc_handle* handle) {
  if (!c || !handle || peer < 0 || peer >= c->plan.world) { set_error("msi_ctx_import: bad argument"); return MSI_EINVAL; }
  if (peer == c->rank) return 0;
  if (c->opened[peer]) return 0;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle->bytes, sizeof(h));
  void* p = nullptr;
  MSI_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  c->peer[peer] = reinterpret_cast<char*>(p);
  c->opened[peer] = true;
  return 0;
}

extern "C" int msi_ctx_finalize(msi_ctx* c) {
  if (!c) { set_error("msi_ctx_finalize: null"); return MSI_EINVAL; }
  const msi_plan& p = c->plan;
  for (int r = 0; r < p.world; ++r)
    if (!c->opened[r]) { set_error("msi_ctx_finalize: peer %d not imported", r); return MSI_ESTATE; }
  DevCtx& d = c->dev;
  memset(&d, 0, sizeof(d));
  d.n_a = p.n_a; d.n_e = p.n_e; d.n_world = p.world; d.E = p.experts; d.K = p.topk;
  d.H = p.hidden; d.Hp = p.inter; d.E_l = plan_el(p); d.slots = p.slots;
  d.max_tokens = p.max_tokens; d.my_a = c->my_a; d.my_e = c->my_e;
  d.tp = plan_tp(p); d.nodes = plan_nodes(p);
  d.my_node = c->my_e >= 0 ? c->my_e / d.tp : -1;
  d.my_tp = c->my_e >= 0 ? c->my_e % d.tp : 0;
  d.cap = c->my_layout.cap;
  d.recv_rows = c->my_layout.recv_rows;
  d.timeout_ns = c->timeout_ns;
  for (int q = 0; q < p.n_e; ++q) {
    const int r = p.expert_ranks[q];
    Layout L = make_layout(p, role_attn(p, r), true);
    d.ecntab_of[q] = reinterpret_cast<uint64_t*>(c->peer[r] + L.cntab);
    d.arrive_of[q] = reinterpret_cast<uint32_t*>(c->peer[r] + L.arrive);
    d.recv_of[q] = c->peer[r] + L.recv;
  }
  for (int s = 0; s < p.n_a; ++s) {
    const int r = p.attn_ranks[s];
    Layout L = make_layout(p, true, role_expert(p, r));
    d.comb_of[s] = reinterpret_cast<uint32_t*>(c->peer[r] + L.comb);
  }
  const Layout& M = c->my_layout;
  d.my_cntab = reinterpret_cast<uint64_t*>(c->heap + M.cntab);
  d.my_arrive = reinterpret_cast<uint32_t*>(c->heap + M.arrive);
  d.my_comb = reinterpret_cast<uint32_t*>(c->heap + M.comb);
  d.my_dticket = reinterpret_cast<uint32_t*>(c->heap + M.dticket);
  d.my_fticket = reinterpret_cast<uint32_t*>(c->heap + M.fticket);
  d.my_ause = reinterpret_cast<uint32_t*>(c->heap + M.ause);
  d.my_euse = reinterpret_cast<uint32_t*>(c->heap + M.euse);
  d.my_status = reinterpret_cast<int32_t*>(c->heap + M.status);
  d.trace = nullptr;
  d.tp_a = plan_tpa(p);
  d.my_tpready = reinterpret_cast<uint32_t*>(c->heap + M.tpready);
  d.my_tprs = reinterpret_cast<uint32_t*>(c->heap + M.tprs);
  d.my_tpuse = reinterpret_cast<uint32_t*>(c->heap + M.tpuse);
  d.my_tpticket = reinterpret_cast<uint32_t*>(c->heap + M.tpticket);
  if (c->attn && d.tp_a > 1) {
    const int node0 = c->my_a / d.tp_a * d.tp_a;
    d.my_ta = c->my_a - node0;
    for (int j = 0; j < d.tp_a; ++j) {
      const int r = p.attn_ranks[node0 + j];
      Layout L = make_layout(p, true, role_expert(p, r));
      d.tpx_of[j] = c->peer[r] + L.tpx;
      d.tprsb_of[j] = c->peer[r] + L.tprsb;
      d.tpready_of[j] = reinterpret_cast<uint32_t*>(c->peer[r] + L.tpready);
      d.tprs_of[j] = reinterpret_cast<uint32_t*>(c->peer[r] + L.tprs);
    }
  }
  MSI_CUDA(cudaMemset(c->heap, 0, M.ctrl_bytes));
  MSI_CUDA(cudaDeviceSynchronize());
  c->finalized = true;
  return 0;
}

extern "C" int msi_ctx_reset(msi_ctx* c) {
  if (!c || !c->finalized) { set_error("msi_ctx_reset: context not finalized"); return MSI_ESTATE; }
  MSI_CUDA(cudaDeviceSynchronize());
  MSI_CUDA(cudaMemset(c->heap, 0, c->my_layout.ctrl_bytes));  // counters, tickets, uses, status, count table
  MSI_CUDA(cudaMemset(c->workspace, 0, c->ws_bytes));
  MSI_CUDA(cudaDeviceSynchronize());
  return 0;
}

extern "C" int msi_ctx_buffer(msi_ctx* c, int which, int slot, void** ptr, size_t* bytes) {
  if (!c || !ptr || !bytes || slot < 0 || slot >= c->plan.slots) { set_error("msi_ctx_buffer: bad argument"); return MSI_EINVAL; }
  const Layout& L = c->my_layout;
  switch (which) {
    case MSI_BUF_RECV:
      if (!c->expert) break;
      *ptr = c->heap + L.recv + slot * L.recv_slot; *bytes = L.recv_slot; return 0;
    case MSI_BUF_HBUF:
      if (!c->expert) break;
      *ptr = c->hbuf; *bytes = (size_t)L.cap * c->plan.inter * 2; return 0;
    case MSI_BUF_TP_X:
      if (!c->attn || plan_tpa(c->plan) < 2) break;
      *ptr = c->heap + L.tpx + slot * L.tpx_slot; *bytes = L.tpx_slot; return 0;
    case MSI_BUF_CNTAB: {
      const size_t per = (size_t)c->plan.n_a * c->plan.experts * 8;
      *ptr = c->heap + L.cntab + slot * per; *bytes = per; return 0;
    }
  }
  set_error("msi_ctx_buffer: buffer %d not present for this rank's role", which);
  return MSI_EINVAL;
}

extern "C" int msi_ctx_workspace(msi_ctx* c, void** ptr, size_t* bytes) {
  if (!c || !ptr || !bytes) { set_error("msi_ctx_workspace: null"); return MSI_EINVAL; }
  *ptr = c->workspace;
  *bytes = c->ws_bytes;
  return 0;
}

extern "C" int msi_poll_status(msi_ctx* c, int32_t* status) {
  if (!c || !status) { set_error("msi_poll_status: null"); return MSI_EINVAL; }
  MSI_CUDA(cudaMemcpy(status, c->heap + c->my_layout.status, sizeof(int32_t), cudaMemcpyDeviceToHost));
  return 0;
}

extern "C" int msi_ctx_stats(msi_ctx* c, uint64_t* rows, uint64_t* calls) {
  if (!c || !rows || !calls) { set_error("msi_ctx_stats: null"); return MSI_EINVAL; }
  uint64_t v[2];
  MSI_CUDA(cudaMemcpy(v, c->heap + c->my_layout.stats, sizeof(v), cudaMemcpyDeviceToHost));
  *rows = v[0];
  *calls = v[1];
  return 0;
}

extern "C" int msi_set_trace(msi_ctx* c, int on) {
  if (!c || !c->finalized) { set_error("msi_set_trace: context not finalized"); return MSI_ESTATE; }
  c->dev.trace = on ? reinterpret_cast<unsigned long long*>(c->heap + c->my_layout.trace) : nullptr;
  if (on) MSI_CUDA(cudaMemset(c->heap + c->my_layout.trace, 0, 32 * sizeof(unsigned long long)));
  return 0;
}

extern "C" int msi_ctx_trace(msi_ctx* c, uint64_t* out, int n) {
  if (!c || !out || n < 0 || n > 32) { set_error("msi_ctx_trace: bad argument"); return MSI_EINVAL; }
  MSI_CUDA(cudaMemcpy(out, c->heap + c->my_layout.trace, n * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  return 0;
}

extern "C" int msi_set_wait_timeout(msi_ctx* c, uint64_t ns) {
  if (!c) { set_error("msi_set_wait_timeout: null"); return MSI_EINVAL; }
  c->timeout_ns = ns;
  c->dev.timeout_ns = ns;
  return 0;
}

extern "C" int msi_dispatch(msi_ctx* c, const void* x, const int32_t* cnt, const int32_t* idx,
                            const int32_t* slot, int T, int mb_slot, uint32_t epoch, void* stream) {
  if (!c || !c->finalized) { set_error("msi_dispatch: context not finalized"); return MSI_ESTATE; }
  if (!c->attn) { set_error("msi_dispatch: rank %d has no attention role", c->rank); return MSI_EINVAL; }
  MSI_REQUIRE(T >= 0 && T <= c->plan.max_tokens, "msi_dispatch: T=%d exceeds max_tokens=%d", T, c->plan.max_tokens);
  MSI_REQUIRE(mb_slot >= 0 && mb_slot < c->plan.slots && epoch != 0xffffffffu, "msi_dispatch: bad slot/epoch");
  MSI_REQUIRE(cnt && (T == 0 || (x && idx && slot)), "msi_dispatch: null pointer");
  const size_t bytes = (size_t)T * c->plan.topk * c->plan.hidden * 2;
  // ~64 KB of row stores per CTA, at most one CTA per SM (rows are split into
  // parts so every warp has work); small micro-batches use few CTAs, which
  // keeps the last-CTA release cheap
  int grid = (int)((bytes + 65535) / 65536);
  grid = grid < 1 ? 1 : (grid > num_sms() ? num_sms() : grid);
  MSI_CUDA(launch_k(dispatch_kernel, dim3(grid), dim3(kDispThreads), 0, reinterpret_cast<cudaStream_t>(stream),
                    c->dev, reinterpret_cast<const __nv_bfloat16*>(x), cnt, idx, slot, T, mb_slot, epoch));
  return check_launch("dispatch_kernel");
}

extern "C" int msi_route_dispatch(msi_ctx* c, const void* x, const void* wg, int T, int E, const int32_t* rep,
                                  int R, int32_t* idx, int32_t* pidx, float* w, int32_t* cnt, int32_t* slot,
                                  int mb_slot, uint32_t epoch, void* stream) {
  if (!c || !c->finalized) { set_error("msi_route_dispatch: context not finalized"); return MSI_ESTATE; }
  if (!c->attn) { set_error("msi_route_dispatch: rank %d has no attention role", c->rank); return MSI_EINVAL; }
  const msi_plan& p = c->plan;
  MSI_REQUIRE(T >= 0 && T <= p.max_tokens, "msi_route_dispatch: T=%d exceeds max_tokens=%d", T, p.max_tokens);
  MSI_REQUIRE(mb_slot >= 0 && mb_slot < p.slots && epoch != 0xffffffffu, "msi_route_dispatch: bad slot/epoch");
  MSI_REQUIRE(rep ? (E >= 1 && E <= p.experts && pidx) : E == p.experts,
              "msi_route_dispatch: E must equal the plan's experts (or its logical count with a replica table)");
  const DevCtx& dv = c->dev;
  DispatchArgs d{};
  d.on = 1;
  d.s = c->my_a;
  d.n_send = p.n_a;
  d.n_e = p.n_e;
  d.E_l = dv.E_l;
  d.tp = dv.tp;
  d.H = p.hidden;
  d.K = p.topk;
  d.P = p.experts;
  d.cap_s = p.max_tokens;
  d.slot_row0 = (long long)mb_slot * dv.recv_rows;
  for (int q = 0; q < p.n_e; ++q) {
    d.recv[q] = dv.recv_of[q];
    d.cntab[q] = dv.ecntab_of[q] + (size_t)mb_slot * p.n_a * p.experts;
    d.arrive[q] = dv.arrive_of[q] + mb_slot * CTR_STRIDE;
  }
  d.ause = dv.my_ause + mb_slot * CTR_STRIDE;
  d.epoch = epoch;
  d.status = dv.my_status;
  d.trace = dv.trace;
  return gate_topk(x, wg, T, p.hidden, E, p.topk, idx, w, cnt, slot, c->workspace, reinterpret_cast<cudaStream_t>(stream),
                   rep, rep ? R : 0, rep ? p.experts : 0, c->my_a, rep ? pidx : nullptr, &d);
}

extern "C" int msi_expert_ffn(msi_ctx* c, const void* w13, const void* w2, int mb_slot,
                              uint32_t epoch, void* stream) {
  if (!c || !c->finalized) { set_error("msi_expert_ffn: context not finalized"); return MSI_ESTATE; }
  if (!c->expert) { set_error("msi_expert_ffn: rank %d has no expert role", c->rank); return MSI_EINVAL; }
  MSI_REQUIRE(mb_slot >= 0 && mb_slot < c->plan.slots , "msi_expert_ffn: bad slot");
  MSI_REQUIRE(w13 && w2, "msi_expert_ffn: null weights");
  const msi_plan& p = c->plan;
  const DevCtx& d = c->dev;
  const Layout& L = c->my_layout;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const size_t tab = (size_t)mb_slot * p.n_a * p.experts;

  const int hp_l = p.inter / d.tp;  // this GPU's slice of h' (expert TP)
  GemmLaunch g1{};
  g1.a = c->heap + L.recv + mb_slot * L.recv_slot;
  g1.a_rows = L.recv_rows;
  g1.p.n_src = p.n_a;      // A rows: runs of the (expert, sender) receive regions
  g1.p.cap_s = p.max_tokens;
  g1.p.a_runs = 1;
  if (c->xcomp && !region_runs_forced()) {
    // several senders: wait for their rows and gather the regions into
    // compact per-expert segments, so every GEMM1 tile is one 128-row box
    int grc = gather_regions(g1.a, d.my_cntab + tab, p.experts, d.my_node * d.E_l, p.n_a, d.E_l, p.max_tokens,
                             p.hidden, c->xcomp, d.my_arrive + mb_slot * CTR_STRIDE, epoch,
                             d.my_euse + mb_slot * CTR_STRIDE, (uint32_t)p.n_a, c->timeout_ns, d.my_status, st);
    if (grc) return grc;
    g1.a = c->xcomp;
    g1.a_rows = L.cap;
    g1.p.n_src = 0;
    g1.p.a_runs = 0;
  }
  g1.b = w13;
  g1.p.E_l = d.E_l;
  g1.p.n_total = 2 * hp_l;
  g1.p.nt = 2 * hp_l / 256;
  g1.p.kdim = p.hidden;
  g1.p.cntab = d.my_cntab + tab;
  g1.p.n_a = p.n_a;
  g1.p.E = p.experts;
  g1.p.e0 = d.my_node * d.E_l;
  g1.p.wait_ctr = d.my_arrive + mb_slot * CTR_STRIDE;
  g1.p.epoch = epoch;  // 0: device-tracked (euse + 1)
  g1.p.epoch_src = d.my_euse + mb_slot * CTR_STRIDE;
  g1.p.wait_mul = (uint32_t)p.n_a;
  g1.p.timeout_ns = c->timeout_ns;
  g1.p.status = d.my_status;
  g1.p.stats = reinterpret_cast<unsigned long long*>(c->heap + L.stats);
  g1.p.trace = d.trace;  // stamps 9 (start), 10 (rows arrived)
  g1.p.trace_slot = 9;
  g1.p.mode = 0;
  g1.p.out = reinterpret_cast<__nv_bfloat16*>(c->hbuf);
  g1.p.out_ld = hp_l;
  g1.p.tile_ctr = d.my_fticket + mb_slot * CTR_STRIDE + 1;  // spare words of the slot's ticket line
  int rc = grouped_gemm_launch(g1, st);
  if (rc) return rc;

  GemmLaunch g2{};
  g2.a = c->hbuf;
  g2.a_rows = L.cap;
  g2.b = w2;
  g2.p.E_l = d.E_l;
  g2.p.n_total = p.hidden;
  g2.p.nt = p.hidden / 256;
  g2.p.kdim = hp_l;
  g2.p.cntab = d.my_cntab + tab;
  g2.p.n_a = p.n_a;
  g2.p.E = p.experts;
  g2.p.e0 = d.my_node * d.E_l;
  g2.p.status = d.my_status;
  g2.p.mode = 1;
  g2.p.out_ld = p.hidden;
  g2.p.out = reinterpret_cast<__nv_bfloat16*>(c->heap + L.recv + mb_slot * L.recv_slot);  // Y over X
  g2.p.n_src = p.n_a;      // virtual row v -> its (expert, sender) region row
  g2.p.cap_s = p.max_tokens;
  g2.p.ticket = d.my_fticket + mb_slot * CTR_STRIDE;
  g2.p.tile_ctr = d.my_fticket + mb_slot * CTR_STRIDE + 2;
  for (int s = 0; s < p.n_a; ++s) g2.p.sig[s] = d.comb_of[s] + mb_slot * CTR_STRIDE;
  g2.p.n_sig = p.n_a;
  g2.p.epoch = epoch;
  g2.p.epoch_src = d.my_euse + mb_slot * CTR_STRIDE;
  g2.p.epoch_store = d.my_euse + mb_slot * CTR_STRIDE;  // last CTA: this use is done
  g2.p.trace = d.trace;  // stamps 13 (GEMM2 start), 14 (release to combine)
  g2.p.trace_slot = 12;
  return grouped_gemm_launch(g2, st);
}

extern "C" int msi_expert_wait(msi_ctx* c, int mb_slot, uint32_t epoch, void* stream) {
  if (!c || !c->finalized) { set_error("msi_expert_wait: context not finalized"); return MSI_ESTATE; }
  if (!c->expert) { set_error("msi_expert_wait: rank %d has no expert role", c->rank); return MSI_EINVAL; }
  MSI_REQUIRE(mb_slot >= 0 && mb_slot < c->plan.slots, "msi_expert_wait: bad slot");
  MSI_CUDA(launch_k(expert_wait_kernel, dim3(1), dim3(1), 0, reinterpret_cast<cudaStream_t>(stream), c->dev,
                    mb_slot, epoch));
  return check_launch("expert_wait_kernel");
}

extern "C" int msi_expert_echo(msi_ctx* c, int mb_slot, uint32_t epoch, void* stream) {
  if (!c || !c->finalized) { set_error("msi_expert_echo: context not finalized"); return MSI_ESTATE; }
  if (!c->expert) { set_error("msi_expert_echo: rank %d has no expert role", c->rank); return MSI_EINVAL; }
  MSI_REQUIRE(mb_slot >= 0 && mb_slot < c->plan.slots , "msi_expert_echo: bad slot");
  MSI_CUDA(launch_k(echo_kernel, dim3(1), dim3(1), 0, reinterpret_cast<cudaStream_t>(stream),
                    c->dev, mb_slot, epoch));
  return check_launch("echo_kernel");
}

// Pull sources of this rank's rows of micro-batch slot mb on every expert GPU.
static CombineSrc combine_src(const msi_ctx* c, int mb_slot, const int32_t* dest, const int32_t* slot) {
  const msi_plan& p = c->plan;
  const DevCtx& d = c->dev;
  CombineSrc src{};
  for (int q = 0; q < p.n_e; ++q) src.y[q] = d.recv_of[q] + (size_t)mb_slot * d.recv_rows * p.hidden * 2;
  src.E_l = d.E_l;
  src.tp = d.tp;
  src.n_send = p.n_a;
  src.s = c->my_a;
  src.cap_s = p.max_tokens;
  src.dest = dest;
  src.slot = slot;
  return src;
}

extern "C" int msi_combine(msi_ctx* c, void* out, const float* w, const int32_t* dest, const int32_t* slot,
                           const void* resid, int T, int mb_slot, uint32_t epoch, void* stream) {
  if (!c || !c->finalized) { set_error("msi_combine: context not finalized"); return MSI_ESTATE; }
  if (!c->attn) { set_error("msi_combine: rank %d has no attention role", c->rank); return MSI_EINVAL; }
  MSI_REQUIRE(T >= 0 && T <= c->plan.max_tokens, "msi_combine: T out of range");
  MSI_REQUIRE(mb_slot >= 0 && mb_slot < c->plan.slots, "msi_combine: bad slot");
  MSI_REQUIRE(T == 0 || (out && w && dest && slot), "msi_combine: null pointer");
  const DevCtx& d = c->dev;
  return launch_combine(combine_src(c, mb_slot, dest, slot), w, resid, out, nullptr, T, c->plan.topk, c->plan.hidden,
                        d.my_comb + mb_slot * CTR_STRIDE, epoch, (uint32_t)c->plan.n_e, d.my_ause + mb_slot * CTR_STRIDE,
                        c->timeout_ns, d.my_status, d.trace, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int msi_gather_y(msi_ctx* c, void* y, const int32_t* dest, const int32_t* slot, int T, int mb_slot,
                            void* stream) {
  if (!c || !c->finalized) { set_error("msi_gather_y: context not finalized"); return MSI_ESTATE; }
  if (!c->attn) { set_error("msi_gather_y: rank %d has no attention role", c->rank); return MSI_EINVAL; }
  MSI_REQUIRE(T >= 0 && T <= c->plan.max_tokens && mb_slot >= 0 && mb_slot < c->plan.slots, "msi_gather_y: bad T/slot");
  MSI_REQUIRE(T == 0 || (y && dest && slot), "msi_gather_y: null pointer");
  if (T == 0) return 0;
  return launch_combine(combine_src(c, mb_slot, dest, slot), nullptr, nullptr, nullptr, y, T, c->plan.topk,
                        c->plan.hidden, nullptr, 0, 0, nullptr, 0, nullptr, nullptr,
                        reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int msi_combine_local(const void* y, const float* w, const void* resid, void* out, int T, int K,
                                 int H, void* stream) {
  MSI_REQUIRE(y && w && out && T >= 0 && K >= 1 && H % 8 == 0, "msi_combine_local: bad argument");
  if (T == 0) return 0;
  CombineSrc src{};
  src.y[0] = reinterpret_cast<const char*>(y);
  src.tp = 1;
  return launch_combine(src, w, resid, out, nullptr, T, K, H, nullptr, 0, 0, nullptr, 0, nullptr, nullptr,
                        reinterpret_cast<cudaStream_t>(stream));
}

// ------------------------------------------------- attention-node TP ----
static int tp_check(msi_ctx* c, const char* fn, int T, int mb_slot) {
  if (!c || !c->finalized) { set_error("%s: context not finalized", fn); return MSI_ESTATE; }
  if (!c->attn || c->dev.tp_a < 2) { set_error("%s: rank %d is not in an attention TP node", fn, c->rank); return MSI_EINVAL; }
  MSI_REQUIRE(T >= 1 && T <= c->plan.max_tokens, "%s: T=%d outside [1, max_tokens=%d]", fn, T, c->plan.max_tokens);
  MSI_REQUIRE(mb_slot >= 0 && mb_slot < c->plan.slots, "%s: bad slot", fn);
  return 0;
}

extern "C" int msi_tp_publish(msi_ctx* c, const void* x, int T, int mb_slot, uint32_t epoch, void* stream) {
  if (int rc = tp_check(c, "msi_tp_publish", T, mb_slot)) return rc;
  (void)epoch;  // every use publishes once: the cumulative ready counter is the epoch
  const DevCtx& d = c->dev;
  const Layout& L = c->my_layout;
  TpSignal sig{};
  sig.ticket = d.my_tpticket + mb_slot * CTR_STRIDE;
  for (int j = 0; j < d.tp_a; ++j) sig.ctr[j] = d.tpready_of[j] + mb_slot * CTR_STRIDE;
  sig.n = d.tp_a;
  char* xin = c->heap + L.tpx + mb_slot * L.tpx_slot;
  return tp_publish(x ? x : xin, xin, T, c->plan.hidden, sig, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int msi_tp_qkv(msi_ctx* c, const void* wqkv_l, int n_heads_l, int n_kv_l, const int32_t* pos, float theta,
                          const int32_t* block_table, int max_pages, void* k_cache, void* v_cache, void* q_out, int T,
                          int mb_slot, uint32_t epoch, void* stream) {
  if (int rc = tp_check(c, "msi_tp_qkv", T, mb_slot)) return rc;
  MSI_REQUIRE(wqkv_l && pos && block_table && k_cache && v_cache && q_out, "msi_tp_qkv: null pointer");
  MSI_REQUIRE(n_kv_l > 0 && n_heads_l > 0 && n_heads_l % n_kv_l == 0, "msi_tp_qkv: bad head counts");
  const int n = (n_heads_l + 2 * n_kv_l) * MSI_HEAD_DIM;
  MSI_REQUIRE(n % 256 == 0, "msi_tp_qkv: n_heads_l + 2 n_kv_l must be even");
  MSI_REQUIRE(theta > 0.f && max_pages > 0, "msi_tp_qkv: bad theta / max_pages");
  const DevCtx& d = c->dev;
  const Layout& L = c->my_layout;
  GemmLaunch g{};
  g.p.a_shards = d.tp_a;
  g.p.E_l = d.tp_a;
  g.p.shard_rows = T;
  for (int j = 0; j < d.tp_a; ++j) g.a_shard[j] = d.tpx_of[j] + mb_slot * L.tpx_slot;
  g.a = g.a_shard[0];
  g.a_rows = T;
  g.b = wqkv_l;
  g.p.n_total = n;
  g.p.nt = n / 256;
  g.p.kdim = c->plan.hidden;
  g.p.mode = 2;
  g.p.pos = pos;
  g.p.rope = rope_inv_table(theta);
  g.p.block_table = block_table;
  g.p.max_pages = max_pages;
  g.p.n_heads = n_heads_l;
  g.p.n_kv = n_kv_l;
  g.p.q_out = reinterpret_cast<__nv_bfloat16*>(q_out);
  g.p.k_cache = reinterpret_cast<__nv_bfloat16*>(k_cache);
  g.p.v_cache = reinterpret_cast<__nv_bfloat16*>(v_cache);
  g.p.wait_ctr = d.my_tpready + mb_slot * CTR_STRIDE;  // every node peer's shard published
  g.p.wait_mul = (uint32_t)d.tp_a;
  g.p.epoch = epoch;
  g.p.epoch_src = d.my_tpuse + mb_slot * CTR_STRIDE;
  g.p.timeout_ns = c->timeout_ns;
  g.p.status = d.my_status;
  g.p.tile_ctr = d.my_tpticket + mb_slot * CTR_STRIDE + 1;
  return grouped_gemm_launch(g, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int msi_tp_oproj(msi_ctx* c, const void* o, const void* wo_l, int k_l, int T, int mb_slot, uint32_t epoch,
                            void* stream) {
  if (int rc = tp_check(c, "msi_tp_oproj", T, mb_slot)) return rc;
  MSI_REQUIRE(o && wo_l && k_l > 0 && k_l % 64 == 0, "msi_tp_oproj: bad arguments");
  const DevCtx& d = c->dev;
  const Layout& L = c->my_layout;
  GemmLaunch g{};
  g.a = o;
  g.a_rows = (int64_t)d.tp_a * T;
  g.b = wo_l;
  g.p.E_l = 1;
  g.p.dense_rows = (long long)d.tp_a * T;
  g.p.n_total = c->plan.hidden;
  g.p.nt = c->plan.hidden / 256;
  g.p.kdim = k_l;
  g.p.mode = 3;
  g.p.shard_rows = T;
  g.p.out_ld = c->plan.hidden;
  for (int j = 0; j < d.tp_a; ++j)  // this GPU's partial slot in peer j's buffer
    g.p.peer_out[j] = reinterpret_cast<__nv_bfloat16*>(d.tprsb_of[j] + mb_slot * L.tprsb_slot + d.my_ta * L.tpx_slot);
  g.p.epoch = epoch;
  g.p.epoch_src = d.my_tpuse + mb_slot * CTR_STRIDE;
  g.p.status = d.my_status;
  g.p.tile_ctr = d.my_tpticket + mb_slot * CTR_STRIDE + 2;
  g.p.ticket = d.my_tpticket + mb_slot * CTR_STRIDE + 3;
  for (int j = 0; j < d.tp_a; ++j) g.p.sig[j] = d.tprs_of[j] + mb_slot * CTR_STRIDE;
  g.p.n_sig = d.tp_a;
  return grouped_gemm_launch(g, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int msi_tp_reduce(msi_ctx* c, const void* resid, void* out, int T, int mb_slot, uint32_t epoch,
                             void* stream) {
  if (int rc = tp_check(c, "msi_tp_reduce", T, mb_slot)) return rc;
  MSI_REQUIRE(resid && out, "msi_tp_reduce: null pointer");
  const DevCtx& d = c->dev;
  const Layout& L = c->my_layout;
  TpWait wt{};
  wt.ctr = d.my_tprs + mb_slot * CTR_STRIDE;
  wt.use = d.my_tpuse + mb_slot * CTR_STRIDE;
  wt.use_store = d.my_tpuse + mb_slot * CTR_STRIDE;
  wt.epoch = epoch;
  wt.timeout_ns = c->timeout_ns;
  wt.status = d.my_status;
  return tp_reduce(resid, out, c->heap + L.tprsb + mb_slot * L.tprsb_slot, (long long)c->plan.max_tokens * c->plan.hidden,
                   d.tp_a, T, c->plan.hidden, wt, reinterpret_cast<cudaStream_t>(stream));
}
