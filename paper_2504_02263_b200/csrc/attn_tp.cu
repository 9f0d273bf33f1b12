// attn_tp.cu -- attention-node tensor parallelism.
//
// An attention node is tp_a GPUs (DeploymentPlan.tp_a).  Each GPU of the node
// owns a token shard of T tokens (its M2N sender batch) and 1/tp_a of the
// heads.  Per layer:
//   publish   x shard -> this GPU's symmetric slot buffer; release every node
//             peer's ready counter                                (this file)
//   QKV       all-gather + GEMM in one kernel: the tcgen05 GEMM loads each
//             peer's shard with its own TMA map straight from the peer's HBM
//             over NVLink, tile by tile (the Flux-style fusion the paper uses,
//             PAPER.md:441-443); epilogue = RoPE + paged-KV append of this
//             GPU's heads for all node tokens          (expert_gemm.cu, a_shards)
//   attention decode attention of this GPU's heads      (attention.cu)
//   O proj    row-parallel GEMM whose epilogue stores each output row into the
//             owning peer's partial buffer over NVLink (the reduce-scatter
//             fused into the epilogue); the last CTA releases the peers'
//             counters                                   (expert_gemm.cu, mode 3)
//   reduce    y = bf16(x + sum_r partial_r) in ascending r          (this file)
// Ordering across GPUs is by cumulative counters per micro-batch slot (epoch
// = the slot's use count, device-tracked): QKV waits ready >= epoch * tp_a,
// reduce waits rs >= epoch * tp_a.  Write-after-read reuse of the shard and
// partial buffers is safe by causality (a GPU republishes slot j only after
// its reduce of j, which needed every peer's O projection of j, which came
// after that peer's QKV read of the shard).
#include <algorithm>

#include "common.cuh"
#include "tp.h"

namespace msi {
namespace {

constexpr int kTpThreads = 256;

// x (T x H bf16) -> xin (this GPU's slot buffer), then the last CTA releases
// every node peer's ready counter.
__global__ void __launch_bounds__(kTpThreads)
tp_publish_kernel(const uint4* __restrict__ x, uint4* __restrict__ xin, long long nvec, TpSignal sig) {
  __shared__ int s_last;
  pdl_trigger();
  pdl_wait();
  if (x != xin)
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nvec; i += (long long)gridDim.x * blockDim.x)
      xin[i] = x[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    s_last = atomicAdd(sig.ticket, 1u) == gridDim.x - 1;
    if (s_last) {
      *sig.ticket = 0;
      fence_sys();
      for (int j = 0; j < sig.n; ++j) red_release_sys_add(sig.ctr[j], 1u);
    }
  }
}

// out[t] = bf16(resid[t] + sum_r part[r][t]) in fp32, ascending r, after
// every node peer's O projection of this use has landed.
__global__ void __launch_bounds__(kTpThreads)
tp_reduce_kernel(const __nv_bfloat16* __restrict__ resid, __nv_bfloat16* __restrict__ out,
                 const __nv_bfloat16* __restrict__ part, long long part_stride, int tp, int T, int H,
                 TpWait wt) {
  __shared__ int s_ok;
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x == 0) {
    uint32_t epoch = resolve_epoch(wt.epoch, wt.use, 1u, wt.status);
    bool ok = epoch != 0 && wait_geq(wt.ctr, epoch * (uint32_t)tp, wt.timeout_ns, wt.status);
    if (ok && blockIdx.x == 0) *(volatile uint32_t*)wt.use_store = epoch;  // read only by later kernels
    s_ok = ok;
  }
  __syncthreads();
  if (!s_ok) return;
  const long long nvec = (long long)T * H / 8;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nvec; i += (long long)gridDim.x * blockDim.x) {
    const uint4 r = reinterpret_cast<const uint4*>(resid)[i];
    float acc[8] = {bf16lo(r.x), bf16hi(r.x), bf16lo(r.y), bf16hi(r.y),
                    bf16lo(r.z), bf16hi(r.z), bf16lo(r.w), bf16hi(r.w)};
    for (int j = 0; j < tp; ++j) {
      const uint4 v = *reinterpret_cast<const uint4*>(part + j * part_stride + i * 8);
      acc[0] += bf16lo(v.x); acc[1] += bf16hi(v.x); acc[2] += bf16lo(v.y); acc[3] += bf16hi(v.y);
      acc[4] += bf16lo(v.z); acc[5] += bf16hi(v.z); acc[6] += bf16lo(v.w); acc[7] += bf16hi(v.w);
    }
    reinterpret_cast<uint4*>(out)[i] = make_uint4(pack_bf16x2(acc[0], acc[1]), pack_bf16x2(acc[2], acc[3]),
                                                  pack_bf16x2(acc[4], acc[5]), pack_bf16x2(acc[6], acc[7]));
  }
}

}  // namespace

int num_sms();

int tp_publish(const void* x, void* xin, int T, int H, const TpSignal& sig, cudaStream_t st) {
  const long long nvec = (long long)T * H / 8;
  const int grid = (int)std::min<long long>(2LL * num_sms(), std::max<long long>(1, (nvec + kTpThreads - 1) / kTpThreads));
  MSI_CUDA(launch_k(tp_publish_kernel, dim3(grid), dim3(kTpThreads), 0, st, reinterpret_cast<const uint4*>(x),
                    reinterpret_cast<uint4*>(xin), nvec, sig));
  return check_launch("tp_publish_kernel");
}

int tp_reduce(const void* resid, void* out, const void* part, long long part_stride, int tp, int T, int H,
              const TpWait& wt, cudaStream_t st) {
  const long long nvec = (long long)T * H / 8;
  const int grid = (int)std::min<long long>(2LL * num_sms(), std::max<long long>(1, (nvec + kTpThreads - 1) / kTpThreads));
  MSI_CUDA(launch_k(tp_reduce_kernel, dim3(grid), dim3(kTpThreads), 0, st,
                    reinterpret_cast<const __nv_bfloat16*>(resid), reinterpret_cast<__nv_bfloat16*>(out),
                    reinterpret_cast<const __nv_bfloat16*>(part), part_stride, tp, T, H, wt));
  return check_launch("tp_reduce_kernel");
}

}  // namespace msi
