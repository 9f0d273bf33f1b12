/*
 * msinfer.h -- C ABI of libmsinfer.so, the B200 (sm_100a) implementation of
 * MegaScale-Infer's disaggregated expert-parallel MoE decode step
 * (arXiv 2504.02263).
 *
 * The reference ships no native entry points for this path (SURVEY.md §0,
 * §8b): its only code is the Python config layer
 * (/root/reference/pkg/src/moeplan/catalog.py), mirrored by
 * paper_2504_02263_b200/config.py.  Each entry point below replaces one
 * operation the paper describes; the citation says which.
 *
 * Conventions (all functions):
 *   - plain pointers and sizes, no C++ or torch types;
 *   - device pointers unless stated; bf16 tensors are passed as void*;
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default);
 *   - every call is asynchronous on `stream` and never synchronizes the host;
 *   - return 0 on success, > 0 = cudaError_t, < 0 = MSI_E* below; the text
 *     of the last error of the calling thread is msi_last_error();
 *   - the caller owns every tensor it passes; the library owns (and frees in
 *     msi_ctx_destroy) the symmetric heap it allocates in msi_ctx_create;
 *   - one host thread per process and per GPU; a context is not re-entrant.
 */
#ifndef MSINFER_H_
#define MSINFER_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MSI_MAX_RANKS 8
#define MSI_IPC_HANDLE_BYTES 64
#define MSI_ROW_ALIGN 128 /* per-expert receive segment alignment (rows) */

enum {
  MSI_EINVAL = -1,      /* bad argument / shape */
  MSI_EARCH = -2,       /* device is not sm_100 */
  MSI_ESTATE = -3,      /* context not finalized / peer missing */
  MSI_ETIMEOUT = -4,    /* a device-side wait exceeded its bound (see msi_poll_status) */
  MSI_EDRIVER = -5      /* CUDA driver entry point unavailable */
};

/* Buffer ids for msi_ctx_buffer (inspection by tests / benches). */
enum {
  MSI_BUF_RECV = 0,   /* expert GPU: received rows [E_l][n_a][max_tokens][H] bf16 per slot
                       * (after the expert FFN: the expert outputs in place) */
  MSI_BUF_HBUF = 3,   /* expert GPU: SwiGLU activations [cap][H'] bf16 (one, shared) */
  MSI_BUF_CNTAB = 4,  /* count table [n_a][E] of (epoch<<32 | count) per slot */
  MSI_BUF_TP_X = 5    /* attention TP: this GPU's token shard [max_tokens][H] bf16 per slot */
};

/* Deployment plan.  Vocabulary of SPEC.md:311 (n_a, m) plus n_e; tp = 1.
 * Expert e lives on expert index e / (experts / n_e) (contiguous blocks). */
typedef struct {
  int32_t world;                         /* ranks (GPUs) in the deployment        */
  int32_t n_a;                           /* attention GPUs (DP replicas)          */
  int32_t n_e;                           /* expert GPUs (EP group)                */
  int32_t attn_ranks[MSI_MAX_RANKS];     /* global rank of attention index s     */
  int32_t expert_ranks[MSI_MAX_RANKS];   /* global rank of expert index q        */
  int32_t hidden;                        /* h   (MoeModelSpec.hidden)             */
  int32_t inter;                         /* h'  (MoeModelSpec.intermediate)       */
  int32_t experts;                       /* E   (MoeModelSpec.experts)            */
  int32_t topk;                          /* K   (MoeModelSpec.topk)               */
  int32_t max_tokens;                    /* b_a: tokens per attention GPU per mb  */
  int32_t slots;                         /* m:   micro-batch slots (ping-pong)    */
  int32_t tp_e;                          /* expert GPUs per expert node (tensor   */
                                         /* parallel over h'; 0 or 1 = none).     */
                                         /* Node j = expert indices [j tp_e,      */
                                         /* (j+1) tp_e); every GPU of a node gets */
                                         /* all of the node's rows and holds h'/  */
                                         /* tp_e features of each local expert;   */
                                         /* the combine sums the tp_e partials.   */
  int32_t tp_a;                          /* attention GPUs per attention node     */
                                         /* (tensor parallel over heads; 0 or 1 = */
                                         /* none).  Node i = attention indices    */
                                         /* [i tp_a, (i+1) tp_a); every GPU keeps */
                                         /* its own max_tokens token shard (its   */
                                         /* M2N batch) and 1/tp_a of the heads.   */
} msi_plan;

typedef struct msi_ctx msi_ctx;

typedef struct {
  unsigned char bytes[MSI_IPC_HANDLE_BYTES];
} msi_ipc_handle;

/* ---- library ------------------------------------------------------------ */
int msi_version(void);
const char* msi_last_error(void);
/* 0 if the current device is sm_100 (B200) and the library's kernels load. */
int msi_check_device(void);

/* ---- context: symmetric heap + peer mapping ("pre-registered
 * tensor"; the M2N library's registration step, here CUDA IPC over NVLink) -- */
int msi_ctx_create(const msi_plan* plan, int rank, msi_ctx** out);
int msi_ctx_destroy(msi_ctx* ctx);
/* IPC handle of this rank's heap, to be exchanged out of band. */
int msi_ctx_export(msi_ctx* ctx, msi_ipc_handle* out);
/* Map peer `peer_rank`'s heap (no-op for own rank). */
int msi_ctx_import(msi_ctx* ctx, int peer_rank, const msi_ipc_handle* handle);
/* After every peer is imported; zeroes the control words (call, then barrier
 * across ranks, before the first dispatch). */
int msi_ctx_finalize(msi_ctx* ctx);
int msi_ctx_buffer(msi_ctx* ctx, int which, int slot, void** ptr, size_t* bytes);
/* Recovery after a device-side wait timed out (MSI_ETIMEOUT, sticky abort
 * flag): synchronizes the device and zeroes this rank's control words (arrival
 * counters, tickets, tile counters, slot use counts, status, count table) and
 * the router workspace.  Every rank of the deployment calls it, then a barrier
 * across ranks, as after msi_ctx_finalize; epochs restart at 1. */
int msi_ctx_reset(msi_ctx* ctx);
/* Device status word: 0 = ok, else a MSI_E* code set by a device-side wait. */
int msi_poll_status(msi_ctx* ctx, int32_t* status);
/* Expert-role counters: rows through msi_expert_ffn and number of calls since
 * msi_ctx_finalize (device-side, exact; read synchronously). */
int msi_ctx_stats(msi_ctx* ctx, uint64_t* rows, uint64_t* calls);
/* Phase tracing (SPEC.md:232 timeline): when on, the kernels
 * write %globaltimer stamps (ns) of this rank's phases into a 32-slot trace
 * line: 0/1/2 dispatch start/counts ready/release, 3/4/5 echo start/rows
 * arrived/release, 6/7/8 combine start/rows arrived/end, 9/10 expert FFN
 * start/rows arrived, 13/14 GEMM2 start/release.  Takes effect for calls
 * (and CUDA-graph captures) made after it. */
int msi_set_trace(msi_ctx* ctx, int on);
int msi_ctx_trace(msi_ctx* ctx, uint64_t* out, int n);
/* Bound on device-side spin waits, in nanoseconds (default 20 s). */
int msi_set_wait_timeout(msi_ctx* ctx, uint64_t ns);
int msi_ctx_workspace(msi_ctx* ctx, void** ptr, size_t* bytes);

/* ---- (1) gate + top-K router, fused with per-expert counts, normalized
 * weights and slot placement -------------
 * x [T,H] bf16, wg [E,H] bf16 (row-major).  Outputs idx [T,K] int32 (descending
 * logit, ties -> lower expert), w [T,K] fp32 (softmax over the K chosen
 * logits), cnt [E] int32, slot [T,K] int32 = rank of token t among this
 * sender's tokens routed to idx[t,k] (ascending token order).  Bit-exact with
 * oracle/msi_oracle.c (pinned fp32 reduction order, deterministic exp).
 * workspace: msi_gate_topk_workspace(T, E) bytes, zero-filled once before the
 * first call (the kernels reset the ticket word they need at zero); for E >= 64
 * it includes a [T][E] fp32 logits scratch (small-T split path).
 * H % 256 == 0, 1 <= K <= min(E,32). */
size_t msi_gate_topk_workspace(int T, int E);
int msi_gate_topk(const void* x, const void* wg, int T, int H, int E, int K,
                  int32_t* idx, float* w, int32_t* cnt, int32_t* slot,
                  void* workspace, void* stream);

/* Router with replicated experts (load balance; SPEC.md
 * balance_experts): rep[e*(R+1)] = replica count of logical expert e,
 * rep[e*(R+1)+1+r] = its r-th physical slot (0 <= slot < P).  Token t of
 * sender `sender` routed to e goes to replica (t + sender) mod count; pidx
 * [T,K] gets the physical slot, cnt [P] and slot [T,K] are per physical slot
 * (idx and w stay logical).  workspace: msi_gate_topk_workspace(T, P). */
int msi_gate_topk_placed(const void* x, const void* wg, int T, int H, int E, int K,
                         const int32_t* rep, int R, int P, int sender, int32_t* idx,
                         int32_t* pidx, float* w, int32_t* cnt, int32_t* slot,
                         void* workspace, void* stream);

/* ---- (1) M2N dispatch (sender; receiver PAPER.md:408-411)
 * Stores each row x[t] over NVLink peer memory into its expert GPU's receive
 * region for (local expert e_l, sender s) -- receive row
 * (e_l * n_a + s) * max_tokens + slot[t,k] of the slot's buffer -- with its
 * (s, t*K+k) metadata; then publishes cnt (this sender's counts, tagged with
 * the epoch) to every expert GPU and releases their arrival counters.  No
 * other sender's counts are needed before the payload moves.  `epoch` counts the
 * uses of `mb_slot` from 1; epoch 0 means "the slot's next use" as counted on
 * the device (msi_dispatch/msi_combine: attention side; msi_expert_ffn /
 * msi_expert_echo: expert side), which makes a whole step capturable in a CUDA
 * graph.  Explicit and device epochs may be mixed: every call records the
 * epoch it used. */
int msi_dispatch(msi_ctx* ctx, const void* x, const int32_t* cnt,
                 const int32_t* idx, const int32_t* slot, int T, int mb_slot,
                 uint32_t epoch, void* stream);

/* ---- (1) fused router + M2N dispatch (top-K, counts,
 * normalized weights and the scatter fused with the gating computation): one
 * launch computes msi_gate_topk's outputs for x [T,H] (wg [E,H]) and stores
 * every routed row into its receive region as msi_dispatch does -- each CTA
 * sends its rows as soon as a decoupled look-back over the CTAs before it
 * fixes their slots; the last CTA publishes the counts and releases the
 * expert GPUs.  rep/R (may be NULL/0): replicated experts as in
 * msi_gate_topk_placed (E = logical experts, the plan's experts = physical
 * slots P, pidx [T,K] receives the physical slot); with rep == NULL, E must
 * equal the plan's experts and pidx may be NULL.  Uses the context's router
 * workspace.  Epoch rules as msi_dispatch. */
int msi_route_dispatch(msi_ctx* ctx, const void* x, const void* wg, int T, int E, const int32_t* rep, int R,
                       int32_t* idx, int32_t* pidx, float* w, int32_t* cnt, int32_t* slot, int mb_slot,
                       uint32_t epoch, void* stream);

/* Block `stream` (one spinning thread, no other SM use) until every sender
 * released `mb_slot`'s epoch -- the wait msi_expert_ffn performs itself --
 * so that the FFN launched after it starts on resident rows and can be timed
 * without the pipeline wait (PAPER.md:408-411 receiver side).  Epoch rules as
 * msi_expert_ffn (pass the same value; 0 = device-tracked). */
int msi_expert_wait(msi_ctx* ctx, int mb_slot, uint32_t epoch, void* stream);
/* ---- (2) expert FFN (SwiGLU): waits for all senders'
 * rows, then two tcgen05/TMEM/TMA grouped GEMMs over the local experts:
 *   H = bf16(silu(X W_gate^T) * (X W_up^T)),  Y = bf16(H W_down^T)
 * whose epilogue stores every Y row over its X in the receive region (local
 * HBM) and releases the attention GPUs, whose combine pulls it (N2M leg,
 * PAPER.md:97).
 * w13: msi_pack_w13 layout [E_l][2H'][H]; w2: [E_l][H][H'] (natural). */
int msi_expert_ffn(msi_ctx* ctx, const void* w13, const void* w2, int mb_slot,
                   uint32_t epoch, void* stream);

/* Identity expert (M2N measurement): waits like msi_expert_ffn and releases
 * the same counters without touching the rows (Y = X in the receive regions,
 * which the combine pulls back).  dispatch + echo + combine is the pure M2N
 * round trip of PAPER.md §5's latency/throughput figures. */
int msi_expert_echo(msi_ctx* ctx, int mb_slot, uint32_t epoch, void* stream);

/* ---- (3) combine (N2M leg PAPER.md:97): waits for all expert
 * GPUs, then pulls the K (x tp_e) expert output rows of every token straight
 * from the expert GPUs' receive regions over NVLink (its own routing names
 * the rows: region (dest % E_l, this sender), row slot) and reduces them:
 * out[t] = bf16(resid[t] + sum_{k,r} w[t,k] * y[t,k,r]) (fp32 fmaf, ascending
 * (k, r); resid may be NULL).  dest/slot: the router's physical slots and
 * slots of this micro-batch (msi_route_dispatch / msi_gate_topk outputs). */
int msi_combine(msi_ctx* ctx, void* out, const float* w, const int32_t* dest, const int32_t* slot,
                const void* resid, int T, int mb_slot, uint32_t epoch, void* stream);
/* The expert output rows themselves, y [T][K * tp_e][H] bf16 (the combine's
 * inputs, for verification; call after the combine of the same use). */
int msi_gather_y(msi_ctx* ctx, void* y, const int32_t* dest, const int32_t* slot, int T, int mb_slot,
                 void* stream);

/* ---- building blocks (also used by tests) -------------------------------- */
/* Expert GEMM variant: 1 = one CTA per 128x256 tile, 2 = CTA pairs
 * (cta_group::2, 256x256 tiles, half pairs for odd 128-row tails), 0 = the
 * default (env MSI_GEMM_CG, else 2).  Process-wide tuning knob. */
int msi_set_gemm_cta_group(int cg);
/* w13[e]: every 256 rows = [gate 64 | up 64 | gate 64 | up 64] of 128
 * consecutive features (matching gate/up in each 128-column half). */
int msi_pack_w13(const void* w_gate, const void* w_up, void* w13, int E_l,
                 int inter, int hidden, void* stream);
/* Stand-alone grouped SwiGLU FFN on compact rows: x [rows][H] where local
 * expert e owns rows [seg_start[e], seg_start[e]+total[e]) with seg_start a
 * MSI_ROW_ALIGN-aligned prefix of total; y [rows][H].  hbuf >= rows x H'. */
int msi_grouped_ffn(const void* x, const int32_t* total, int E_l, int rows,
                    const void* w13, const void* w2, void* hbuf, void* y,
                    int hidden, int inter, void* stream);
/* Stand-alone combine on a local [T,K,H] buffer (no waits). */
int msi_combine_local(const void* y, const float* w, const void* resid,
                      void* out, int T, int K, int H, void* stream);
/* ---- Attention stage: GQA decode over paged KV.
 * The reference models it as T_a = k1*b_a + k2 with the KV traffic
 * 2*b*s*h*bytes/g (Table 3).
 *
 * Paged KV cache (per layer): k_cache / v_cache bf16
 *   [num_pages][n_kv][MSI_KV_PAGE][MSI_HEAD_DIM]
 * block_table int32 [T][max_pages] (page ids of sequence t, in order).
 * Query heads n_heads = G * n_kv, G <= 16; head h uses KV head h / G. */
#define MSI_KV_PAGE 64
#define MSI_HEAD_DIM 128

/* RoPE (rotate-half, base theta) on the new token's q and k at position
 * pos[t], then append k, v into the cache slot (page block_table[t][pos/64],
 * row pos%64).  qkv bf16 [T][qkv_ld] holds q (n_heads*128) | k (n_kv*128) |
 * v (n_kv*128); q_out bf16 [T][n_heads*128] receives the rotated q. */
int msi_rope_append(const void* qkv, int64_t qkv_ld, const int32_t* pos, int T,
                    int n_heads, int n_kv, float theta,
                    const int32_t* block_table, int max_pages,
                    void* k_cache, void* v_cache, int64_t num_pages,
                    void* q_out, void* stream);
/* The expert FFN on (expert, sender) receive regions without a context (the
 * layout msi_expert_ffn reads; tests and A/B runs): region (e, s) of cap_s
 * rows at row (e*n_src + s)*cap_s of x_reg, cntab [n_src][E_l] uint64 with
 * the region's row count in the low 32 bits.  a_runs = 1: GEMM1 loads each
 * 128-row tile as runs of the regions (one power-of-two TMA box per piece).
 * xcomp != NULL (>= hbuf_rows x hidden): the regions are first gathered into
 * compact 128-aligned per-expert segments of xcomp and GEMM1 reads those
 * (msi_expert_ffn's path when several senders share an expert).  Y of every
 * row is stored at its own row of y_reg (may alias x_reg).  hbuf >=
 * hbuf_rows x inter, hbuf_rows >= sum over experts of the 128-rounded totals. */
int msi_grouped_ffn_regions(const void* x_reg, const uint64_t* cntab, int n_src,
                            int64_t cap_s, int E_l, const void* w13, const void* w2,
                            void* hbuf, int64_t hbuf_rows, void* y_reg, int hidden,
                            int inter, int a_runs, void* xcomp, void* stream);
/* ---- attention-node tensor parallelism (plan.tp_a > 1)
 * Per layer and micro-batch slot, on every attention GPU of a node, in this
 * order on one stream (epoch 0 = device-tracked, as for the M2N calls):
 *   msi_tp_publish  x shard [T][H] -> this GPU's symmetric shard buffer, then
 *                   release the node peers (x may be that buffer itself:
 *                   msi_ctx_buffer(MSI_BUF_TP_X)).
 *   msi_tp_qkv      all-gather fused into the QKV GEMM: the tcgen05 GEMM
 *                   reads every peer's shard over NVLink with its own TMA
 *                   map; wqkv_l = this GPU's [q heads | k heads | v heads]
 *                   rows [(n_heads_l + 2 n_kv_l) 128][H]; epilogue = RoPE +
 *                   paged-KV append for all tp_a*T node tokens (node token
 *                   s*T + t = peer s's token t), q_out [tp_a*T][n_heads_l][128].
 *   (msi_decode_attention over this GPU's heads, o [tp_a*T][n_heads_l*128])
 *   msi_tp_oproj    row-parallel O projection, wo_l = W_o[:, this GPU's head
 *                   columns] [H][n_heads_l*128]; the epilogue stores each
 *                   token's partial row into its owner's partial buffer over
 *                   NVLink (reduce-scatter fused into the GEMM).
 *   msi_tp_reduce   out[t] = bf16(resid[t] + sum_r partial_r[t]) (fp32, r
 *                   ascending) once every peer's partials landed.
 * T <= max_tokens, the same T on every GPU of the node. */
int msi_tp_publish(msi_ctx* ctx, const void* x, int T, int mb_slot, uint32_t epoch,
                   void* stream);
int msi_tp_qkv(msi_ctx* ctx, const void* wqkv_l, int n_heads_l, int n_kv_l, const int32_t* pos,
               float theta, const int32_t* block_table, int max_pages, void* k_cache,
               void* v_cache, void* q_out, int T, int mb_slot, uint32_t epoch, void* stream);
int msi_tp_oproj(msi_ctx* ctx, const void* o, const void* wo_l, int k_l, int T, int mb_slot,
                 uint32_t epoch, void* stream);
int msi_tp_reduce(msi_ctx* ctx, const void* resid, void* out, int T, int mb_slot, uint32_t epoch,
                  void* stream);

/* The attention stage's two projections (Table 3, "QKV
 * Project" and "Attn Output") on the expert GEMM's tcgen05 kernel, run as
 * one dense "expert" of T rows (CTA-pair 256x256 tiles, TMA, TMEM).
 * tile_ctr: a caller-owned zeroed uint32 in device memory (the launch's
 * dynamic tile counter; each call leaves it at 0; one in-flight call per
 * counter).
 *
 * out[t][0:N] = bf16(a[t] . b[0:N]^T (+ resid[t][0:N])) -- a bf16 [T][K],
 * b bf16 [N][K] (K-major), N % 256 == 0, K % 64 == 0, fp32 accumulation and
 * one rounding (the residual is added in fp32). */
int msi_dense_gemm(const void* a, int64_t T, const void* b, int N, int K,
                   void* out, int64_t out_ld, const void* resid, int64_t resid_ld,
                   uint32_t* tile_ctr, void* stream);
/* fp32 out[t][e] = x[t] . wg[e] on the tensor cores (the router's candidate
 * pass for fine-grained MoE; accumulation order of the MMA, not the pinned
 * one): E % 256 == 0, H % 64 == 0. */
int msi_dense_logits(const void* x, int64_t T, const void* wg, int E, int H, float* out,
                     uint32_t* tile_ctr, void* stream);
/* QKV projection with RoPE and the paged-KV append in the GEMM epilogue:
 * qkv = bf16(x . wqkv^T) (wqkv bf16 [(n_heads + 2 n_kv) 128][hidden]), then
 * exactly what msi_rope_append does with that qkv -- q heads rotated into
 * q_out [T][n_heads][128], k heads rotated and v heads copied into the cache
 * slot (page block_table[t][pos[t]/64], row pos[t]%64).  No qkv buffer. */
int msi_qkv_rope_append(const void* x, int64_t T, int hidden, const void* wqkv,
                        int n_heads, int n_kv, const int32_t* pos, float theta,
                        const int32_t* block_table, int max_pages,
                        void* k_cache, void* v_cache, void* q_out,
                        uint32_t* tile_ctr, void* stream);
/* Workspace bytes msi_decode_attention needs for T sequences (split-KV
 * partials; 0 when no split is used). */
size_t msi_decode_attention_workspace(int T, int n_heads, int n_kv, int max_pages);
/* out[t][h*128 + d] = softmax(q[t,h] . K[t,kvh]^T * scale) V[t,kvh], over
 * seq_lens[t] cached tokens; out bf16 [T][n_heads*128]. */
int msi_decode_attention(const void* q, const void* k_cache, const void* v_cache,
                         int64_t num_pages, const int32_t* block_table, int max_pages,
                         const int32_t* seq_lens, int T, int n_heads, int n_kv,
                         float scale, void* out, void* workspace, size_t ws_bytes,
                         void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MSINFER_H_ */
