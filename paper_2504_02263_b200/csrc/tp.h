// tp.h -- attention-node tensor parallelism kernels (attn_tp.cu) as seen by m2n.cu.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/msinfer.h"

namespace msi {

// Release one counter on each node peer (last CTA of the launch).
struct TpSignal {
  uint32_t* ticket;                 // this GPU's last-CTA ticket word (0 at rest)
  uint32_t* ctr[MSI_MAX_RANKS];     // peers' counters of the slot
  int n;
};

// Wait for ctr >= epoch * tp (epoch 0: *use + 1), then store the use.
struct TpWait {
  const uint32_t* ctr;
  const uint32_t* use;
  uint32_t* use_store;
  uint32_t epoch;
  uint64_t timeout_ns;
  int32_t* status;
};

int tp_publish(const void* x, void* xin, int T, int H, const TpSignal& sig, cudaStream_t st);
int tp_reduce(const void* resid, void* out, const void* part, long long part_stride, int tp, int T, int H,
              const TpWait& wt, cudaStream_t st);

}  // namespace msi
