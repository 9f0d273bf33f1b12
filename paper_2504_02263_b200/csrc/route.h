// route.h -- the fused router + M2N dispatch (router.cu) as seen by m2n.cu.
//
// PAPER.md:444-447 fuses top-K, per-expert counts, normalized weights and the
// scatter of tokens to their experts with the gating computation.  Here that
// is one kernel: each CTA routes its tokens, learns the rank of its tokens
// among the sender's earlier ones by a decoupled look-back over the CTAs
// before it (no second pass, no last-CTA scan), and stores its rows straight
// into the expert GPUs' receive regions; the last CTA to finish publishes the
// sender's counts and releases the receivers' arrival counters.
#pragma once

#include <stdint.h>

#include "../../include/msinfer.h"

namespace msi {

// Receive layout (per expert GPU, per micro-batch slot): one region of cap_s
// rows per (local expert e_l, sender s), at row (e_l * n_send + s) * cap_s,
// so a sender's rows need no other sender's counts (cap_s = max_tokens: a
// sender routes each token to an expert at most once).
struct DispatchArgs {
  int on;                            // 0: router only
  int s, n_send;                     // this sender's index, senders (n_a)
  int n_e, E_l, tp;                  // expert GPUs, physical slots per expert node, GPUs per node
  int H, K, P;                       // hidden, top-K, physical expert slots
  long long cap_s;                   // rows per (expert, sender) region
  long long slot_row0;               // first row of micro-batch slot mb in recv
  char* recv[MSI_MAX_RANKS];         // per expert index q
  uint64_t* cntab[MSI_MAX_RANKS];    // per expert index q: [n_send][P] of slot mb
  uint32_t* arrive[MSI_MAX_RANKS];   // per expert index q: arrival counter of slot mb
  uint32_t* ause;                    // this sender's use counter of slot mb
  uint32_t epoch;                    // 0: device-tracked (ause + 1)
  int32_t* status;
  unsigned long long* trace;         // stamps 0 (start) / 2 (release) when tracing
};

// Router (+ dispatch when d && d->on).  rep == nullptr: P = E.
int gate_topk(const void* x, const void* wg, int T, int H, int E, int K, int32_t* idx, float* w, int32_t* cnt,
              int32_t* slot, void* ws, cudaStream_t st, const int32_t* rep = nullptr, int R = 0, int P = 0,
              int sender = 0, int32_t* pidx = nullptr, const DispatchArgs* d = nullptr);
size_t gate_topk_workspace(int T, int E);

}  // namespace msi
