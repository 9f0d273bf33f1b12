// gemm.h -- launch interface of the grouped expert GEMM (expert_gemm.cu).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/msinfer.h"
#include "common.cuh"

#define MSI_MAX_LOCAL_EXPERTS 256  /* DeepSeek-V3 shape on one GPU */
#define MSI_SMALL_LOCAL_EXPERTS 64 /* GEMM variant with the deeper pipeline */

namespace msi {

struct GemmParams {
  int E_l;        // local experts
  int n_total;    // B rows per expert (2H' for GEMM1, H for GEMM2)
  int nt;         // N tiles per expert (n_total / 256)
  int kdim;       // reduction dim (H for GEMM1, H' for GEMM2)
  // segment sizes: explicit device array, or summed from the count table
  const int32_t* totals;    // [E_l] or null
  const uint64_t* cntab;    // [n_a][E] of (epoch << 32 | count), used when totals == null
  int n_a, E, e0;           // e0 = first global expert of this GPU
  // optional wait before any load (GEMM1 on an expert GPU)
  const uint32_t* wait_ctr;
  uint32_t epoch;             // 0: read *epoch_src + 1 on the device
  const uint32_t* epoch_src;  // this slot's expert-side use counter
  uint32_t wait_mul;          // wait for *wait_ctr >= epoch * wait_mul
  uint32_t* epoch_store;      // optional: last CTA stores the epoch (use done)
  uint64_t timeout_ns;
  int32_t* status;          // [0] = error code, [1] = abort flag
  unsigned long long* stats;  // optional: [0] += rows processed, [1] += 1 (one CTA)
  unsigned long long* trace;  // optional %globaltimer stamps: [slot] start,
  int trace_slot;             //   [slot+1] rows arrived, [slot+2] release
  // epilogue
  int mode;                 // 0: SwiGLU -> out[row][out_ld]; 1: plain bf16 rows; 2: QKV + RoPE/append;
                            // 3: plain rows to peer_out (attention-TP reduce-scatter);
                            // 4: fp32 rows (router logits)
  __nv_bfloat16* out;       // mode 0: hbuf; mode 1: y (n_src > 0: the receive
                            //   regions themselves -- Y of a row replaces its X,
                            //   which the attention GPU's combine pulls)
  int out_ld;               // elements per output row (H' or H)
  // dynamic tile scheduler: CTAs (pairs) take tiles in order from this
  // counter (0 at launch; the launch's last fetch resets it)
  uint32_t* tile_ctr;
  // half-pair tiles load A with the 64-row box (set by the launcher)
  int a64;
  // TMA loads with L2 eviction priorities (set by the launcher)
  int l2hint;
  int pfb;  // > 0: L2 prefetch of the B (weight) tile this many k-blocks ahead (MSI_GEMM_PFB)
  // receive regions (msi_expert_ffn): counts per (sender, expert) from cntab;
  // virtual row v of expert e lives in region (e, s) of cap_s rows at offset
  // v - pre[e][s].  a_runs = 1: GEMM1 loads A by runs of those regions; the
  // mode 1 epilogue stores row v there.  n_src = 0: compact rows.
  int n_src;
  long long cap_s;
  int a_runs;
  // completion signal (last CTA): red.release.sys +1 on each sig[i]
  uint32_t* ticket;
  uint32_t* sig[MSI_MAX_RANKS];
  int n_sig;
  // dense GEMMs of the attention stage (E_l = 1, rows = dense_rows, no
  // segment table): mode 1 adds resid[row][resid_ld] before the bf16
  // rounding (O projection + residual); mode 2 is the QKV projection with
  // RoPE on q/k heads and the paged-KV append in the epilogue (msi_qkv_rope_append)
  long long dense_rows;
  const __nv_bfloat16* resid;
  long long resid_ld;
  const int32_t* pos;          // mode 2: position of row t's new token
  const int32_t* block_table;  // mode 2: [rows][max_pages]
  int max_pages, n_heads, n_kv;
  RopeInv rope;                // mode 2: theta^(-2i/128) (rope_inv_table)
  __nv_bfloat16* q_out;        // [rows][n_heads][128]
  __nv_bfloat16* k_cache;      // [pages][n_kv][64][128]
  __nv_bfloat16* v_cache;
  // attention TP (msi_tp_qkv / msi_tp_oproj): a_shards > 0 -> "expert" e is
  // node peer e's token shard of shard_rows rows, loaded from its own tensor
  // map (am.m[e], the peer's symmetric buffer) at the shard's rows; every
  // shard uses the same B (shared weights); output row = e * shard_rows + r.
  // mode 3: output row t goes to peer_out[t / shard_rows] at row
  // t % shard_rows (the O projection's reduce-scatter over NVLink).
  int a_shards;
  int shard_rows;
  // split-K (mode 4): ksplit planes of plane floats each, summed by the reader
  int ksplit;
  long long plane;
  __nv_bfloat16* peer_out[MSI_MAX_RANKS];
};

struct GemmLaunch {
  const void* a;   // [a_rows][kdim] bf16
  int64_t a_rows;
  const void* b;   // [E_l * n_total][kdim] bf16
  int grid;        // 0 = one CTA per SM
  int cta_group;   // 1: 128x256 tiles per CTA; 2: 256x256 tiles per CTA pair; 0 = default
  const void* a_shard[MSI_MAX_RANKS];  // p.a_shards > 0: shard e's A ([a_rows][kdim] each)
  GemmParams p;
};

int grouped_gemm_launch(const GemmLaunch& L, cudaStream_t st);
int num_sms();
// Rows of the (expert, sender) receive regions -> compact 128-aligned
// per-expert segments of xc (GEMM1's A when several senders share an
// expert); wait_ctr != null: first wait for *wait_ctr >= epoch * wait_mul.
int dense_logits_f32(const void* x, int64_t rows, const void* wg, int E, int H, float* out, uint32_t* tile_ctr,
                     cudaStream_t st, int ksplit);
int gather_regions(const void* recv, const uint64_t* cntab, int E, int e0, int n_src, int E_l, long long cap_s,
                   int H, void* xc, const uint32_t* wait_ctr, uint32_t epoch, const uint32_t* epoch_src,
                   uint32_t wait_mul, uint64_t timeout_ns, int32_t* status, cudaStream_t st);

}  // namespace msi
