/*
 * nosa_b200.h — C ABI of the B200-native NOSA offloaded sparse-attention decode step.
 *
 * The reference (arXiv 2510.13602 testbench, /root/reference/pkg/src/nosa_sim) has no FFI:
 * everything is in-process NumPy.  Each entry point below is the batched, device-resident
 * replacement of one reference call site; the citation names the reference interface it
 * stands behind (file:line under pkg/src/nosa_sim/).  A Python maintainer binds this header
 * with ctypes; paper_2510_13602_b200/_lib.py is that binding.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Device pointers are CUDA device addresses; `stream`
 *    arguments are cudaStream_t handles passed as void* (NULL = legacy default stream).
 *  - Every call returns an int status (NOSA_OK or one NOSA_ERR_*); the message of the last
 *    failure is nosa_last_error(ctx) (ctx may be NULL for creation failures).
 *  - Single writer per context, one context per GPU.  All per-step calls are asynchronous
 *    on the caller's stream; calls named nosa_read_* synchronise and copy to host memory.
 *  - Errors raised inside kernels (CapacityExceeded, ...) are latched in a device flag word
 *    and surfaced by nosa_check_errors() / the next synchronising call.
 */
#ifndef NOSA_B200_H
#define NOSA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: the reference's exception types (kv_manager.py:31-56, config.py:38-65) ---- */
#define NOSA_OK 0
#define NOSA_ERR_VALUE 1         /* ValueError: shapes / config / argument range          */
#define NOSA_ERR_CAPACITY 2      /* kv_manager.CapacityExceeded  (kv_manager.py:47-48)    */
#define NOSA_ERR_UNKNOWN_KEY 3   /* kv_manager.UnknownKey        (kv_manager.py:43-44)    */
#define NOSA_ERR_OUT_OF_BLOCKS 4 /* kv_manager.OutOfBlocks       (kv_manager.py:35-36)    */
#define NOSA_ERR_CUDA 5          /* CUDA runtime failure (RuntimeError)                    */
#define NOSA_ERR_STATE 6         /* call order misuse, e.g. step before prefill            */

/* device error-flag bits (nosa_check_errors) */
#define NOSA_FLAG_CAPACITY 1u
#define NOSA_FLAG_EMPTY_SUPPORT 2u /* softmax over empty support (numerics.py:50-52)       */
#define NOSA_FLAG_NOT_RESIDENT 4u  /* all-resident run met a miss that is not a newborn block      */
#define NOSA_FLAG_FULL 8u          /* append past the head capacity (HeadState, decode.py:65-71); refused */

/* selectors (decode.py:28 SELECTORS) */
#define NOSA_SELECTOR_NOSA 0     /* selection.nosa_select      (selection.py:130-160)     */
#define NOSA_SELECTOR_INFLLMV2 1 /* selection.infllmv2_select  (selection.py:163-178)     */

/* eviction-head variants (attention.py:26 VARIANTS; `retaining` needs hidden states and is
 * out of scope on this path) */
#define NOSA_VARIANT_ED_DMA 0 /* beta = s_e_c                (attention.py:160-161)       */
#define NOSA_VARIANT_S_DMA 1  /* beta = 0                    (attention.py:164-165)       */
#define NOSA_VARIANT_DMA 2    /* beta = log(mean exp-score)  (attention.py:162-164)       */

#define NOSA_DTYPE_BF16 0
#define NOSA_DTYPE_FP32 1

#define NOSA_GATHER_UVA 0     /* zero-copy SM gather kernel over mapped pinned memory     */
#define NOSA_GATHER_MEMCPY 1  /* copy-engine path: host-planned, one cudaMemcpyAsync a block */
#define NOSA_GATHER_TMA 2     /* TMA bulk copies pinned host -> shared -> HBM slot         */
#define NOSA_GATHER_HOSTPACK 3 /* host threads pack the misses, one DMA per 2 MiB chunk      */
#define NOSA_GATHER_HYBRID 4   /* units split: host-packed DMAs + the SM gather, concurrently */

/* AttentionConfig (config.py:15-36) plus the engine extents of one GPU. */
typedef struct NosaConfig {
  int32_t n, d, n_head, n_kv_head, d_head, n_b, n_s, n_w, k, k_q, k_e;
  int32_t accounting; /* 0 = "inclusive", 1 = "exclusive" (config.py:8-12)             */
  int32_t batch;      /* sequences owned by this context                                */
  int32_t layers;     /* attention layers (independent caches)                          */
  int32_t max_tokens; /* per-sequence cache capacity in tokens (HeadState capacity)     */
  int32_t fast_slots; /* HBM slots per (layer, sequence, kv head) = fast-tier num_blocks */
  int32_t dtype;      /* NOSA_DTYPE_*: K/V/q storage type                               */
  int32_t variant;    /* NOSA_VARIANT_*                                                 */
  int32_t residency;  /* NOSA_RESIDENCY_*                                               */
  int32_t attend_chunk; /* KV blocks per split-K attention work item (1..8); 0 = auto from
                           the batch size.  Outputs are bit-identical for a fixed value.    */
  int32_t attend_layers; /* layers per persistent attention launch in the pipelined schedule;
                            0 = auto (8 when every block fits in HBM, else 1)               */
  int32_t exact_scan;    /* 0: screened selection (bf16 pre-scan of the pool, f64 rescoring of
                            the candidates: the same picks as a full f64 scan); 1: full f64  */
  int32_t slow_tier_device; /* -1: slow tier in pinned host memory (PCIe); >= 0: in that GPU's
                               HBM, read by peer access over NVLink (the context's own device =
                               loopback, for single-GPU testing)                                */
} NosaConfig;

/* residency contract */
#define NOSA_RESIDENCY_PER_SEQUENCE 0 /* one manager per (layer, sequence, head): SURVEY §8a   */
#define NOSA_RESIDENCY_SHARED 1       /* one fast pool of batch*fast_slots per (layer, head)
                                         shared by the batch, planned in batch order: the
                                         reference simulator (offload_sim.py:254-299)          */

/* ResidencyStats (kv_manager.py:101-122), summed over a (layer, sequence, head) range. */
typedef struct NosaStats {
  int64_t hits, misses, new_blocks, evictions, steps;
  int64_t bytes_up, bytes_down; /* misses * bytes_per_block, evictions * bytes_per_block */
  int64_t candidates;           /* pool rows rescored in f64 by the screened selector     */
  int64_t topk_required;        /* required blocks from the selection pool (top-k picks)  */
  int64_t topk_misses;          /* fetches among them: hit_rate_topk = 1 - misses/required
                                   (offload_sim.py:291-293)                                */
} NosaStats;

/* Per-step inputs/outputs of nosa_decode_step: one pointer per tensor, layer-major.
 *   q     [layers][batch][n_head][d_head]     (dtype)
 *   k_new [layers][batch][n_kv_head][d_head]  (dtype)
 *   v_new [layers][batch][n_kv_head][d_head]  (dtype)
 *   out   [layers][batch][n_head][d_head]     (float32)                                 */
typedef struct NosaStepIO {
  const void* q;
  const void* k_new;
  const void* v_new;
  float* out;
  int32_t selector;    /* NOSA_SELECTOR_* */
  int32_t gather_mode; /* NOSA_GATHER_*   */
  int32_t schedule;    /* 0 = layer-pipelined (gather of layer l overlaps scoring of l+1..),
                          1 = layer-serial (select of layer l+1 after layer l completes) */
} NosaStepIO;

/* nosa_decode_step_host: the same tensors in HOST memory (pinned for asynchronous copies;
 * pageable works but serialises).  Same layouts and meanings as NosaStepIO. */
typedef struct NosaHostStepIO {
  const void* q;
  const void* k_new;
  const void* v_new;
  float* out;
  int32_t selector;
  int32_t gather_mode;
  int32_t schedule;
} NosaHostStepIO;

/* nosa_decode_step_hidden: hidden states in (the reference's DecodeEngine.step(h_t) input),
 * q/k/v projected on the GPU by the weights of nosa_set_projection.
 *   h   [layers][batch][d]               (bf16, device)
 *   out [layers][batch][n_head][d_head]  (float32, device)                                    */
typedef struct NosaHiddenStepIO {
  const void* h;
  float* out;
  int32_t selector;
  int32_t gather_mode;
  int32_t schedule;
} NosaHiddenStepIO;

typedef struct NosaCtx NosaCtx;

/* ---- configuration ---------------------------------------------------------------- */

/* AttentionConfig.__post_init__ validation (config.py:38-65) plus engine-extent checks.
 * Writes the ValueError text into msg. */
int nosa_config_validate(const NosaConfig* cfg, char* msg, int msg_len);

/* Derived budgets (config.py:72-94): blocks_q, blocks_e, blocks_topk. */
int nosa_config_budgets(const NosaConfig* cfg, int32_t* blocks_q, int32_t* blocks_e,
                        int32_t* blocks_topk);

/* ---- context lifetime ------------------------------------------------------------- */

/* Allocates the HBM slot pools (PhysicalLayout FAST, kv_manager.py:59-81), the block tables
 * (TieredBlockManager.__init__, kv_manager.py:138-167) and the pinned, mapped host mirror
 * (the SLOW tier).  Every logical block starts in the slow tier (offload_sim.py:262-266). */
int nosa_ctx_create(const NosaConfig* cfg, int device, NosaCtx** out);
void nosa_ctx_destroy(NosaCtx* ctx);
const char* nosa_last_error(const NosaCtx* ctx);
/* bytes of device and pinned host memory held by the context */
int nosa_ctx_memory(const NosaCtx* ctx, int64_t* device_bytes, int64_t* host_bytes);

/* EvictionHead weights (attention.py:104-118): w1 (d_head x n_head) row-major, w2 (n_head),
 * host float64.  Required before nosa_prefill for ed-dma / s-dma / dma. */
int nosa_set_eviction_head(NosaCtx* ctx, const double* w1, const double* w2);

/* ---- prefill / run start (DecodeEngine.prefill, start_run: decode.py:139-150) ------- */

/* Caches t tokens for sequences [seq_begin, seq_begin+seq_count) of one layer and makes
 * them slow-resident.  k, v: device [seq_count][n_kv_head][t][d_head] (dtype).  Computes the
 * per-token importance scores (importance_scores, attention.py:121-146), the block means
 * used for selection (compress_blocks, attention.py:42-59) and writes the host mirror.
 * Resets the sequences' residency to all-slow.  Synchronous w.r.t. `stream` completion
 * of its inputs only. */
int nosa_prefill(NosaCtx* ctx, int layer, int seq_begin, int seq_count, const void* k,
                 const void* v, int t, void* stream);

/* nosa_prefill, then every cached block is also made fast-resident: block i of each
 * (sequence, head) in slot i, as TieredBlockManager.allocate(FAST, ...) in block order
 * (kv_manager.py:171-183).  The all-resident configuration; needs fast_slots >= blocks,
 * else NOSA_ERR_CAPACITY. */
int nosa_prefill_resident(NosaCtx* ctx, int layer, int seq_begin, int seq_count, const void* k,
                          const void* v, int t, void* stream);

/* BlockGeometry.for_run (selection.py:46-50) for every layer of the sequences: freezes
 * recent_start at the current cache length and ranks the frozen pool by its query-agnostic
 * score (the second phase of nosa_select, selection.py:151-156). */
int nosa_start_run(NosaCtx* ctx, int seq_begin, int seq_count, void* stream);

/* ---- the hot path, stage by stage (DecodeEngine.step decode.py:152-190 +
 *      the residency loop of simulate_decode offload_sim.py:279-299) -------------------- */

/* K1+K2 fused: GQA-summed scoring of the frozen pool (decode.py:171-172), top-k selection
 * (nosa_select / infllmv2_select), required = fixed U topk (offload_sim.py:233-234), then
 * plan_transfers + apply_transfers on the block tables (kv_manager.py:205-279).
 * q: device [batch][n_head][d_head] (dtype).  Enqueues the layer's miss list. */
int nosa_select_plan(NosaCtx* ctx, int layer, const void* q, int selector, void* stream);

/* K1 only (no residency change): fills the selection buffers read by nosa_read_selection. */
int nosa_select(NosaCtx* ctx, int layer, const void* q, int selector, void* stream);

/* K2 only, with caller-provided required block sets (TieredBlockManager.plan_transfers +
 * apply_transfers, kv_manager.py:205-279).  req: device int32 [batch][n_kv_head][fast_slots],
 * n_req: device int32 [batch][n_kv_head]; each row sorted ascending, unique. */
int nosa_cache_plan(NosaCtx* ctx, int layer, const int32_t* req, const int32_t* n_req,
                    void* stream);

/* K3: moves the layer's missed blocks from the host mirror into their HBM slots
 * (the `mover` of apply_transfers, kv_manager.py:290, 300-305). */
int nosa_gather(NosaCtx* ctx, int layer, int mode, void* stream);

/* K4+K5: block-sparse biased attention over the required blocks (attend_biased over the
 * token mask, attention.py:167-182, decode.py:179-185), then append of the new token with its
 * importance score (decode.py:187-189).  out: device float32 [batch][n_head][d_head]. */
int nosa_attend(NosaCtx* ctx, int layer, const void* q, const void* k_new, const void* v_new,
                float* out, void* stream);

/* All layers of one decode step, pipelined: select+plan on `stream`, the miss gathers on the
 * context's copy stream overlapped with scoring of the next layers, attention after each
 * attention batch's gathers.  Equivalent to per-layer nosa_select_plan, nosa_gather, nosa_attend. */
int nosa_decode_step(NosaCtx* ctx, const NosaStepIO* io, void* stream);

/* nosa_decode_step on host buffers: the reference's own calling convention
 * (DecodeEngine.step takes and returns host arrays, decode.py:152-190), batched.  Each
 * selection group's q/k/v are staged from pinned host memory by an SM zero-copy kernel on the
 * context's input stream ahead of that group's selection (NOSA_STAGE_COPIES=1: copy-engine
 * copies instead); layer l's output comes back on a device->host stream as soon as layer l is
 * done (overlapping later layers).  Asynchronous on
 * `stream`: the host buffers must stay valid, and `out` is complete, once `stream` reaches this
 * point (cudaStreamSynchronize).  The context owns the device staging. */
int nosa_decode_step_host(NosaCtx* ctx, const NosaHostStepIO* io, void* stream);

/* The QKV projection of one layer for nosa_decode_step_hidden (project_qkv, attention.py:67-90;
 * DecodeEngine.step decode.py:162-164): w_t = [W_q | W_k | W_v]^T, device bf16 [n][d],
 * n = (n_head + 2 n_kv_head) d_head, nq = n_head d_head, nk = n_kv_head d_head.  The weights are
 * copied into the context (all layers side by side, so a selection group's projections run as
 * one launch).  bf16 storage only. */
int nosa_set_projection(NosaCtx* ctx, int layer, const void* w_t, int d, int n, int nq, int nk);

/* All layers of one decode step from hidden states: per selection group, the tcgen05
 * projection of its layers (on the selection stream), then the step of nosa_decode_step on
 * the projected q / k / v.  Same schedule, movers and results as nosa_decode_step fed with
 * those q / k / v.  Graph form: nosa_step_graph_capture_hidden + nosa_step_graph_launch. */
int nosa_decode_step_hidden(NosaCtx* ctx, const NosaHiddenStepIO* io, void* stream);
int nosa_step_graph_capture_hidden(NosaCtx* ctx, const NosaHiddenStepIO* io);

/* nosa_decode_step_hidden with HOST buffers (DecodeEngine.step(h_t), decode.py:152-190, calling
 * convention): io->h [layers][batch][d] bf16 and io->out [layers][batch][n_head][d_head] f32 in
 * host memory (pinned: the SMs stage each selection group's hidden states with zero-copy loads;
 * pageable: cudaMemcpyAsync), outputs copied back per attention batch as in
 * nosa_decode_step_host.  Asynchronous on `stream` like nosa_decode_step_host. */
int nosa_decode_step_hidden_host(NosaCtx* ctx, const NosaHiddenStepIO* io, void* stream);

/* CUDA-graph form of nosa_decode_step_host (device movers only: uva / tma): capture once on
 * pinned host buffers; every launch may pass other pinned buffers of the same shapes (the
 * graph's input-staging and output-copy nodes are re-pointed before the launch). */
int nosa_step_graph_capture_host(NosaCtx* ctx, const NosaHostStepIO* io);
int nosa_step_graph_launch_host(NosaCtx* ctx, const NosaHostStepIO* io, void* stream);

/* CUDA-graph form of nosa_decode_step for fixed io pointers: capture once, replay per step. */
int nosa_step_graph_capture(NosaCtx* ctx, const NosaStepIO* io);
int nosa_step_graph_launch(NosaCtx* ctx, void* stream);

/* ---- QKV projection (project_qkv, attention.py:67-90; DecodeEngine.step decode.py:162-164) --- */

/* [q | k | v] = h · w_tᵀ on the tensor cores (tcgen05, fp32 accumulation in TMEM), rounded to bf16.
 * h: device bf16 [m][k] (hidden states, row-major); w_t: device bf16 [n][k] (the columns of
 * [W_q | W_k | W_v], each stored K-contiguous); q/k_out/v: device bf16 [m][nq], [m][nk],
 * [m][n - nq - nk].  K is cut into `splits` (1..8) ranges computed by one thread-block cluster
 * and summed through distributed shared memory in rank order (deterministic).
 * Needs n % 128 == 0 and k % (64 * splits) == 0. */
int nosa_project_qkv(const void* h, int m, int k, const void* w_t, int n, int nq, int nk, void* q,
                     void* k_out, void* v, int splits, void* stream);

/* fp32 form of the projection for fp32 caches (project_qkv, attention.py:67-90, the parity
 * mode): out [m][n] = h [m][k] . w [k][n], device float32, row-major, CUDA-core FMAs in k
 * order.  No context; asynchronous on `stream`. */
int nosa_project_f32(const float* h, int m, int k, const float* w, int n, float* out, void* stream);

/* ---- standalone selector (drop-in for nosa_select / infllmv2_select on given scores) --- */

/* n_prob independent selections.  s_q, s_e: device float64 [n_prob][stride] block scores.
 * pool_lo/pool_hi: device int32 [n_prob] (BlockGeometry.pool_blocks).  Outputs sorted
 * ascending block ids: out_q [n_prob][m_q], out_e [n_prob][m_e], counts n_q/n_e [n_prob].
 * selector NOSA_SELECTOR_INFLLMV2 ignores s_e and uses m_q as the total top-k budget. */
int nosa_select_scores(int n_prob, const double* s_q, const double* s_e, int stride,
                       const int32_t* pool_lo, const int32_t* pool_hi, int m_q, int m_e,
                       int selector, int32_t* out_q, int32_t* n_q, int32_t* out_e,
                       int32_t* n_e, void* stream);

/* ---- readback / statistics (synchronising) ---------------------------------------- */

/* Last selection of a layer, host buffers sized [batch][n_kv_head][cap]:
 * blocks_q/e (sorted), required (sorted, = fixed U topk) and counts.
 * s_q (optional, may be NULL): [batch][n_kv_head][max_blocks] float64 pool scores. */
int nosa_read_selection(NosaCtx* ctx, int layer, int cap, int32_t* blocks_q, int32_t* n_q,
                        int32_t* blocks_e, int32_t* n_e, int32_t* required, int32_t* n_req,
                        double* s_q);

/* Last TransferPlan of a layer (kv_manager.py:84-98), host [batch][n_kv_head][fast_slots]:
 * fetch (block ids, plan order), evict (victims, LRR order), hit counts. */
int nosa_read_plan(NosaCtx* ctx, int layer, int32_t* fetch, int32_t* n_fetch, int32_t* evict,
                   int32_t* n_evict, int32_t* n_hit);

/* Block table of one (layer, sequence, head): slot_of [max_blocks] (-1 = slow tier),
 * block_of [fast_slots] (-1 = free).  TieredBlockManager.lookup / fast_resident. */
int nosa_read_residency(NosaCtx* ctx, int layer, int seq, int head, int32_t* slot_of,
                        int32_t* block_of);

/* Selection scores of the frozen pool, host float64 [batch][n_kv_head][max_blocks]:
 * s_e_c block means (compress_scores) as used by the selector. */
int nosa_read_block_scores(NosaCtx* ctx, int layer, double* s_e_c);

/* Cached K/V of one (layer, sequence, head), host [t][d_head] in dtype, from the host
 * mirror (the slow tier always holds every block; HBM slots hold copies). */
int nosa_read_kv(NosaCtx* ctx, int layer, int seq, int head, int t, void* k, void* v);
/* Copy of one HBM slot, host [2][n_b][d_head] in dtype (un-swizzled). */
int nosa_read_slot(NosaCtx* ctx, int layer, int seq, int head, int slot, void* kv);

int nosa_read_stats(NosaCtx* ctx, int layer_begin, int layer_end, int seq_begin, int seq_end,
                    NosaStats* out);
int nosa_reset_stats(NosaCtx* ctx, void* stream);
/* cache length per (layer, sequence) (HeadState.t, decode.py:70) */
int nosa_read_lengths(NosaCtx* ctx, int32_t* t /* [layers][batch] */);
/* synchronises; returns NOSA_ERR_CAPACITY etc. if a kernel latched an error, and clears it */
int nosa_check_errors(NosaCtx* ctx, uint32_t* flags);

/* Device timing of every kernel of subsequent eager steps, bracketed by CUDA events on the
 * stream each kernel runs on (bench evidence).  Kinds: 0 = select+plan (K1+K2), 1 = gather (K3),
 * 2 = attention (K4, split-K records), 3 = finalize (K4 log-sum-exp merge + K5 append),
 * 4 = host->device input copy and 5 = device->host output copy of nosa_decode_step_host,
 * 6 = QKV projection of nosa_decode_step_hidden.
 * enable(0) turns it off; read synchronises and returns the summed milliseconds and launch
 * counts per kind since enable. */
int nosa_timing_enable(NosaCtx* ctx, int max_launches);
int nosa_timing_read(NosaCtx* ctx, double* total_ms /* [7] */, int64_t* launches /* [7] */);

/* The timed launches since enable, in issue order: kind and start/end milliseconds relative to
 * the first one (a device timeline of the step's streams).  Synchronises. */
int nosa_timing_trace(NosaCtx* ctx, int cap, int32_t* kind, float* start_ms, float* end_ms,
                      int32_t* n);

/* Diagnostics: device-clock (%globaltimer) span of each attention launch, first CTA start to
 * last CTA end, indexed by the launch's first layer; read returns microseconds of the last
 * launch per layer (0 = none) and resets.  Both synchronise. */
int nosa_ktime_enable(NosaCtx* ctx, int on);
int nosa_ktime_read(NosaCtx* ctx, double* span_us /* [layers] */);

/* Diagnostics: cycles spent per phase of the selection kernel, summed over CTAs (cycles[15] =
 * CTAs).  Phases: 1 q_sum, 2 screen scan, 3 radix threshold, 4 f64 rescoring, 5 ranking,
 * 6 NOSA walk, 7 outputs + required list, 8 hit test, 9 victims, 11 apply + writes.
 * Reads (if cycles != NULL) then resets (on = 1) or disables (on = 0).  Synchronises. */
int nosa_select_profile(NosaCtx* ctx, int on, double* cycles /* [16] */);

/* ---- TieredBlockManager (kv_manager.py:130-363): the reference's exclusive two-tier block
 *      manager with its tables, free lists, recency clock and payload in device memory -------- */

/* One manager: per head, `fast_blocks` FAST slots (PhysicalLayout(FAST, ...)) and `slow_blocks` SLOW
 * slots (PhysicalLayout(SLOW, ...)), LIFO free lists initialised [N-1 .. 0] (kv_manager.py:147-150).
 * Keys are dense per-head ids in [0, fast_blocks + slow_blocks) chosen by the caller (the Python
 * binding maps the reference's (batch, head, block) tuples onto them).  store_payload: FAST payload
 * in HBM, SLOW payload in pinned host memory, (num_blocks, heads, 2, n_b, d_head) per tier. */
typedef struct NosaMgr NosaMgr;
int nosa_mgr_create(int heads, int fast_blocks, int slow_blocks, int n_b, int d_head, int element_width,
                    int store_payload, int device, NosaMgr** out);
void nosa_mgr_destroy(NosaMgr* mgr);
const char* nosa_mgr_last_error(const NosaMgr* mgr);
/* allocate (kv_manager.py:171-183): tier 0 FAST / 1 SLOW; NOSA_ERR_OUT_OF_BLOCKS, NOSA_ERR_VALUE
 * (DuplicateKey) */
int nosa_mgr_allocate(NosaMgr* mgr, int tier, int head, int id, int batch, int block, int32_t* slot);
/* free_block (kv_manager.py:185-194): NOSA_ERR_UNKNOWN_KEY */
int nosa_mgr_free(NosaMgr* mgr, int head, int id);
/* plan_transfers (kv_manager.py:205-259) for (batch, head): ids of the required keys in ascending
 * block order (-1 = a key mapped in no tier).  Ticks the clock and stamps last_required like the
 * reference; changes no table.  Outputs fetch ids (required order) and evict ids
 * (least-recently-required order by (last_required, batch, block)).  NOSA_ERR_CAPACITY,
 * NOSA_ERR_UNKNOWN_KEY. */
int nosa_mgr_plan(NosaMgr* mgr, int head, int batch, const int32_t* ids, int n, int32_t* fetch, int32_t* n_fetch,
                  int32_t* evict, int32_t* n_evict, int32_t* hits);
/* plan_transfers with a caller-supplied eviction_policy (kv_manager.py:133-138, 236-250): the same
 * clock tick, recency stamps, fetch ids and hits as nosa_mgr_plan, but no victim choice. When
 * evictions are needed (*shortfall > 0), `candidates` receives the ids of the evictable FAST keys
 * (every FAST key of the head but this call's required ones, in fast-slot order) for the caller's
 * policy to order; the caller takes the first *shortfall of its order (CapacityExceeded when the
 * policy returns fewer). `candidates` holds fast_blocks ids. */
int nosa_mgr_plan_policy(NosaMgr* mgr, int head, int batch, const int32_t* ids, int n, int32_t* fetch,
                         int32_t* n_fetch, int32_t* shortfall, int32_t* candidates, int32_t* n_cand, int32_t* hits);
/* last_required clock of every id of a head ([fast_blocks + slow_blocks]; 0 = never required),
 * the reference's `last_required` map handed to an eviction policy */
int nosa_mgr_recency(NosaMgr* mgr, int head, uint32_t* last);
/* apply_transfers' moves (kv_manager.py:276-298): evictions FAST -> SLOW then fetches SLOW -> FAST,
 * one _move at a time; copy_payload: the default mover's payload copies, on the device.
 * moves (optional): [n_evict + n_fetch][2] source and destination slot of each move (-1, -1 =
 * no-op move). */
int nosa_mgr_apply(NosaMgr* mgr, int head, const int32_t* evict, int n_evict, const int32_t* fetch, int n_fetch,
                   int copy_payload, int32_t* moves);
/* lookup (kv_manager.py:185-190): tier (-1 unmapped, 0 FAST, 1 SLOW) and slot of one key */
int nosa_mgr_lookup(NosaMgr* mgr, int head, int id, int32_t* tier, int32_t* slot);
/* tier / slot of every id of a head ([fast_blocks + slow_blocks] each): dump_table_csv */
int nosa_mgr_tables(NosaMgr* mgr, int head, int8_t* tier, int32_t* slot);
/* the per-head LIFO free lists (bottom to top: the last entry is popped next), as kv_manager.free */
int nosa_mgr_free_lists(NosaMgr* mgr, int head, int32_t* fast, int32_t* n_fast, int32_t* slow, int32_t* n_slow);
/* audit (kv_manager.py:341-363): *bad = 0 when every (tier, head) slot partition holds */
int nosa_mgr_audit(NosaMgr* mgr, int32_t* bad);
/* write_block / read_block (kv_manager.py:305-321): one block's payload, host [2][n_b][d_head] */
int nosa_mgr_block(NosaMgr* mgr, int head, int id, void* data, int write);

/* ---- seeded synthetic inputs (bench / parity tests; not part of the decode step) --------- */

/* Counter-based N(0,1) draws (Irwin-Hall sum of four 16-bit hash fields, times `scale` in fp32),
 * a pure function of (seed, kind, layer, global sequence, head, position, dim): any shard or
 * subset of the batch draws the same bits as paper_2510_13602_b200/workload.py's NumPy twin.
 * kind: 0 prefix K, 1 prefix V, 2 initial query state, 3 query innovations, 4 k_new, 5 v_new.
 * out: device [n_layers][n_seq][heads][n_pos][d] in dtype (bf16: round to nearest even). */
int nosa_synth_normal(uint64_t seed, int kind, int layer0, int n_layers, int seq0, int n_seq, int heads,
                      long long pos0, long long n_pos, int d, float scale, int dtype, void* out, void* stream);

/* One AR(1) query step over state [n_layers][n_seq][heads][d] (float32, device, in place):
 * q_out = round(state); state = fl32(fl32(rho * state) + fl32(sigma * eps)), eps = the kind-3
 * draws at position `step` times `scale`. */
int nosa_synth_ar1_step(uint64_t seed, int layer0, int n_layers, int seq0, int n_seq, int heads, long long step,
                        int d, float rho, float sigma, float scale, float* state, int dtype, void* q_out,
                        void* stream);

/* kernel launches issued by this library since context creation (bench evidence) */
int64_t nosa_launch_count(const NosaCtx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* NOSA_B200_H */
