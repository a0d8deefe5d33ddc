// nosa_ctx.cu — the C ABI (include/nosa_b200.h): context lifetime, the per-layer stages,
// the pipelined multi-layer decode step (+ CUDA graph), readback and statistics.
#include <sys/mman.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <chrono>
#include <thread>
#include <vector>
#if defined(__x86_64__)
#include <immintrin.h>
#endif

#include "../../include/nosa_b200.h"
#include "nosa_device.cuh"

namespace nosa {
cudaError_t launch_select_plan(const Dev& dv, int layer, const void* q, int selector, int mode,
                               const int* ext_req, const int* ext_nreq, cudaStream_t st, int layers = 1);
cudaError_t launch_start_run(const Dev& dv, int seq_begin, int seq_count, cudaStream_t st);
cudaError_t launch_screen_build(const Dev& dv, int seq_begin, int seq_count, cudaStream_t st);
cudaError_t launch_score_readback(const Dev& dv, int layer, cudaStream_t st);
cudaError_t launch_plan_shared(const Dev& dv, int layer, const int* ext_req, const int* ext_nreq, cudaStream_t st);
cudaError_t launch_select_scores(int n_prob, const double* s_q, const double* s_e, int stride,
                                 const int* lo, const int* hi, int m_q, int m_e, int selector,
                                 int* out_q, int* n_q, int* out_e, int* n_e, cudaStream_t st);
cudaError_t launch_gather(const Dev& dv, int layer, cudaStream_t st, int grid, bool tma, int nl = 1);
cudaError_t launch_born(const Dev& dv, int layer, cudaStream_t st, int grid);
cudaError_t launch_scatter(const char* stage, void* const* dst, int count, int bpb, cudaStream_t st);
cudaError_t launch_stage_inputs(const void* const* src, void* const* dst, const size_t* bytes, int grid,
                                cudaStream_t st);
const void* stage_inputs_kernel_fn();
cudaError_t launch_project(const void* A, const void* Bt, int M, int N, int K, int splits, void* q, void* k, void* v,
                           int nq, int nk, cudaStream_t st, int layers = 1);
cudaError_t launch_project_f32(const float* h, const float* w, int M, int K, int N, float* out, cudaStream_t st);

cudaError_t launch_prefill(const Dev& dv, int layer, int seq_begin, int S, const void* k,
                           const void* v, int t, char* staging, cudaStream_t st);
cudaError_t launch_make_resident(const Dev& dv, int layer, int seq_begin, int S, int nblk, cudaStream_t st);
cudaError_t launch_unswizzle(const char* src, char* dst, int nblocks, int n_b, int D, int elem,
                             cudaStream_t st);
cudaError_t launch_attend(const Dev& dv, int layer, int nl, const void* q, const void* kn, const void* vn,
                          float* out, cudaStream_t st, int num_sms);
cudaError_t launch_finalize(const Dev& dv, int layer, const void* kn, const void* vn, float* out, cudaStream_t st,
                            int nl = 1);
bool attend_supported(int n_b, int d_head, int dtype);
bool attend_f32_per_layer();
}  // namespace nosa

using nosa::Dev;

static inline void cpu_relax() {
#if defined(__x86_64__)
  _mm_pause();
#endif
}

// Host threads of the host-pack mover (NOSA_GATHER_HOSTPACK): each job copies `count` blocks of
// `bytes` from scattered host addresses into one contiguous pinned staging buffer.  The caller
// takes part; workers claim blocks with tickets from one 64-bit counter (job generation in the
// high half, block index in the low half), so a ticket always names the job it belongs to and a
// late worker of an earlier job can neither take nor count a block of the next one.  Job
// descriptors alternate between two slots (a job starts only after the previous one is done).
// Workers spin between jobs, sleeping once idle for ~10 ms (e.g. between steps).
struct PackPool {
  struct Job {
    char* const* src = nullptr;
    char* dst = nullptr;
    int count = 0;
    size_t bytes = 0;
  };
  std::vector<std::thread> th;
  Job job[2];
  std::atomic<unsigned long long> next{0};
  std::atomic<unsigned> gen{0};
  std::atomic<int> done{0};
  std::atomic<bool> stop{false};
  void work() {
    for (;;) {
      const unsigned long long t = next.fetch_add(1, std::memory_order_acq_rel);
      const Job& j = job[(t >> 32) & 1];
      const int i = (int)(unsigned)t;
      if (i >= j.count) break;
      memcpy(j.dst + (size_t)i * j.bytes, j.src[i], j.bytes);
      done.fetch_add(1, std::memory_order_release);
    }
  }
  void worker() {
    unsigned seen = gen.load(std::memory_order_acquire);
    long idle = 0;
    while (!stop.load(std::memory_order_relaxed)) {
      const unsigned g = gen.load(std::memory_order_acquire);
      if (g != seen) {
        seen = g;
        work();
        idle = 0;
      } else if (++idle < 200000) {
        cpu_relax();
      } else {
        std::this_thread::sleep_for(std::chrono::microseconds(50));
      }
    }
  }
  void start(int n) {
    for (int i = 0; i < n; ++i) th.emplace_back([this] { worker(); });
  }
  void run(char* const* s, char* d, int n, size_t b) {
    const unsigned g = gen.load(std::memory_order_relaxed) + 1;
    job[g & 1] = Job{s, d, n, b};
    done.store(0, std::memory_order_relaxed);
    next.store((unsigned long long)g << 32, std::memory_order_release);
    gen.store(g, std::memory_order_release);
    work();
    while (done.load(std::memory_order_acquire) < n) cpu_relax();
  }
  ~PackPool() {
    stop = true;
    for (auto& t : th) t.join();
  }
};

struct NosaCtx {
  NosaConfig cfg{};
  Dev dv{};
  int device = 0;
  int num_sms = 148;
  int gather_grid = 8;       // UVA gather CTAs: enough bytes in flight for the link, few SMs taken
  int tma_gather_grid = 24;  // TMA gather CTAs (one warp, 4 x 32 KiB stages each)
  cudaStream_t copy_stream = nullptr;
  cudaStream_t sel_stream = nullptr;  // selections (forked from the caller's stream per step)
  cudaStream_t att_stream = nullptr, att_stream2 = nullptr, fin_stream = nullptr;  // attention (even /
  // odd layers, so one layer's attention tail overlaps the next) and finalize stages
  bool two_att = true;
  std::vector<cudaEvent_t> ev_plan, ev_gather, ev_att, ev_fin;
  cudaEvent_t ev_fork = nullptr;
  char* host_mirror = nullptr;
  size_t host_bytes = 0;
  bool host_registered = false;  // mmap + cudaHostRegister (else cudaHostAlloc)
  int mirror_device = -1;        // >= 0: the slow tier lives in this GPU's HBM (peer tier)
  std::vector<void*> dev_allocs;
  size_t dev_bytes = 0;
  char* staging = nullptr;
  size_t staging_bytes = 0;
  bool have_evhead = false;
  cudaGraph_t graph = nullptr, graph_timed = nullptr;              // clean / instrumented step
  cudaGraphExec_t graph_exec = nullptr, graph_exec_timed = nullptr;
  cudaStream_t capture_stream = nullptr;
  int graph_kernels = 0;
  struct Timed { cudaEvent_t a, b; int kind; };
  std::vector<Timed> timing;       // pre-created event pairs
  size_t timing_used = 0;
  // graph capture of the timing scopes: placeholder events and the event-record nodes
  bool capturing = false;
  std::vector<Timed> cap_events;
  size_t cap_used = 0;
  struct EvNode { cudaGraphNode_t node; int slot; int end; };
  std::vector<EvNode> ev_nodes;
  bool nodes_on_pool = false;  // the nodes currently point at timing-pool events
  std::atomic<long long> launches{0};
  std::string err;
  // copy-engine gather (NOSA_GATHER_MEMCPY): pinned readback of the miss list + batch arrays
  cudaStream_t meta_stream = nullptr;
  int* h_cnt = nullptr;
  int4* h_list = nullptr;
  std::vector<void*> b_dst, b_src;
  // exported copy lists (Dev::x_*): mapped pinned host arrays the planner fills on the device
  void** h_xsrc = nullptr;
  void** h_xdst = nullptr;
  int* h_xcnt = nullptr;
  // host-pack mover (NOSA_GATHER_HOSTPACK): pack threads, pinned host ring -> device ring (one DMA
  // per chunk on the copy stream), scatter kernels on their own stream; dst list in device memory
  PackPool* pack = nullptr;
  int pack_chunk = 64;                 // blocks per chunk (2 MiB at 32 KiB blocks)
  int pack_slots = 8;                  // ring depth
  char* hp_host = nullptr;             // [slots][chunk][bpb] pinned
  char* hp_dev = nullptr;              // [slots][chunk][bpb]
  void** hp_xdst = nullptr;            // [L][B*H*C] device: slot address of every packed block
  std::vector<cudaEvent_t> hp_ev_dma, hp_ev_sc;
  std::vector<char> hp_used;
  int hp_next = 0;
  cudaStream_t scatter_stream = nullptr;
  int hp_split = 1024;                 // this step's host-pack share of the units (of 1024)
  cudaStream_t smg_stream = nullptr;   // hybrid mover: the SM gather's own stream
  std::vector<cudaEvent_t> ev_smg;     // hybrid: SM gather of the attention batch ending at layer l
  // host-buffer step (nosa_decode_step_host): device staging of the step's inputs and outputs,
  // per-layer input-arrival / output-ready events, and the device->host stream
  cudaStream_t d2h_stream = nullptr, in_stream = nullptr;
  std::vector<cudaEvent_t> ev_in;
  std::vector<std::pair<int, int>> groups;  // selection groups (first layer, layers) of the step
  cudaEvent_t ev_d2h = nullptr;
  char* io_buf = nullptr;
  char* hid_buf = nullptr;  // [L][B][d] bf16 device copy of host hidden states (nosa_decode_step_hidden_host)
  size_t hid_bytes = 0;
  size_t io_bytes = 0;
  int stage_grid = 32;              // CTAs of the input-staging kernel (host-buffer step)
  bool stage_with_copies = false;   // NOSA_STAGE_COPIES: stage host inputs with cudaMemcpyAsync
  int attend_layers = 1;            // most layers in one attention launch (pipelined schedule)
  std::vector<int> att_plan;        // layers per attention launch, in order (sums to L)
  std::vector<int> att_l0;          // (per step) first layer of the batch closed at layer l, else -1
  // QKV projection of nosa_decode_step_hidden: per-layer [W_q | W_k | W_v]^T, bf16 [n][d] (caller-owned)
  char* proj_wbuf = nullptr;         // [L][n][d] bf16, the layers' weights side by side
  std::vector<char> proj_set;        // per layer: weights loaded
  int proj_d = 0;
  int step_kernels = 0;             // kernels launched by the last enqueued step
  std::vector<char> prefilled_resident;  // [L][B]: the last prefill of (layer, seq) placed every block in HBM
  int memcpy_born_launches = 0;     // born-block kernels of the copy-engine mover (this step)
  bool select_per_layer = false;
  // graph of the host-buffer step and its host-address nodes (kind 0 = staging kernel, 1 = D2H copy)
  cudaGraph_t graph_host = nullptr;
  cudaGraphExec_t graph_exec_host = nullptr;
  int graph_host_kernels = 0;
  struct HostNode { cudaGraphNode_t node; int kind; };
  std::vector<HostNode> host_nodes;
  const char* cap_hs[3] = {nullptr, nullptr, nullptr};
  const char* cur_hs[3] = {nullptr, nullptr, nullptr};
  float* cap_out = nullptr;
  float* cur_out = nullptr;  // NOSA_SELECT_PER_LAYER: one selection launch per layer
};

// brackets one launch with timing events when timing is enabled (eager steps only)
// During graph capture the same scope records into placeholder events as external event-record
// nodes; every replay re-points those nodes at fresh events of the timing pool, so a graph
// replay is timed per kernel exactly like an eager step.
struct TimeScope {
  NosaCtx* ctx;
  cudaStream_t st;
  NosaCtx::Timed* slot = nullptr;
  bool capture = false;
  TimeScope(NosaCtx* c, cudaStream_t s, int kind, bool on) : ctx(c), st(s) {
    if (ctx->capturing) {
      if (ctx->cap_used < ctx->cap_events.size()) {
        slot = &ctx->cap_events[ctx->cap_used++];
        slot->kind = kind;
        capture = true;
        cudaEventRecordWithFlags(slot->a, st, cudaEventRecordExternal);
      }
    } else if (on && ctx->timing_used < ctx->timing.size()) {
      slot = &ctx->timing[ctx->timing_used++];
      slot->kind = kind;
      cudaEventRecord(slot->a, st);
    }
  }
  ~TimeScope() {
    if (!slot) return;
    if (capture) cudaEventRecordWithFlags(slot->b, st, cudaEventRecordExternal);
    else cudaEventRecord(slot->b, st);
  }
};

static thread_local std::string g_create_error;

static int fail(NosaCtx* ctx, int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (ctx) ctx->err = buf; else g_create_error = buf;
  return code;
}

#define CUDA_TRY(ctx, expr)                                                                   \
  do {                                                                                       \
    cudaError_t _e = (expr);                                                                 \
    if (_e != cudaSuccess) {                                                                 \
      cudaGetLastError(); /* a non-sticky error must not leak into the next call */          \
      return fail(ctx, NOSA_ERR_CUDA, "%s failed: %s", #expr, cudaGetErrorString(_e));       \
    }                                                                                        \
  } while (0)

static int budgets(const NosaConfig& c, int* bq, int* be, int* bt) {
  const int k_e_topk = c.accounting == 0 ? c.k - c.n_s - c.n_w - c.k_q : c.k_e;  // config.py:72-77
  *bq = c.k_q / c.n_b;
  *be = k_e_topk / c.n_b;
  *bt = *bq + *be;
  return NOSA_OK;
}

extern "C" int nosa_config_validate(const NosaConfig* c, char* msg, int msg_len) {
  auto bad = [&](const char* fmt, auto... args) {
    if (msg && msg_len > 0) snprintf(msg, msg_len, fmt, args...);
    return NOSA_ERR_VALUE;
  };
  if (!c) return bad("config is NULL");
  // AttentionConfig.__post_init__ (config.py:38-65), same order and messages
  if (c->n_b <= 0) return bad("n_b must be positive");
  if (c->k != c->k_q + c->k_e) return bad("k must equal k_q + k_e (%d != %d + %d)", c->k, c->k_q, c->k_e);
  const char* names[5] = {"n_s", "n_w", "k", "k_q", "k_e"};
  const int vals[5] = {c->n_s, c->n_w, c->k, c->k_q, c->k_e};
  for (int i = 0; i < 5; ++i) {
    if (vals[i] < 0) return bad("%s must be non-negative", names[i]);
    if (vals[i] % c->n_b != 0) return bad("%s=%d must be divisible by n_b=%d", names[i], vals[i], c->n_b);
  }
  if (!(c->n_s + c->n_w <= c->k && c->k <= c->n))
    return bad("need n_s + n_w <= k <= n, got n_s+n_w=%d, k=%d, n=%d", c->n_s + c->n_w, c->k, c->n);
  if (c->n_head <= 0 || c->n_kv_head <= 0 || c->n_head % c->n_kv_head != 0)
    return bad("n_head=%d must be a positive multiple of n_kv_head=%d", c->n_head, c->n_kv_head);
  if (c->d_head <= 0 || c->d <= 0) return bad("d and d_head must be positive");
  if (c->accounting != 0 && c->accounting != 1) return bad("accounting must be one of ('inclusive', 'exclusive')");
  if (c->accounting == 0 && c->k - c->n_s - c->n_w - c->k_q < 0)
    return bad("inclusive accounting needs k_q <= k - n_s - n_w (k_q=%d, k - n_s - n_w = %d)", c->k_q,
               c->k - c->n_s - c->n_w);
  // engine extents (B200 build)
  if (c->batch <= 0 || c->layers <= 0) return bad("batch and layers must be positive");
  if (c->max_tokens <= 0) return bad("max_tokens must be positive");
  if (c->fast_slots <= 0) return bad("fast_slots must be positive");
  if (c->attend_chunk < 0 || c->attend_chunk > 8) return bad("attend_chunk must be in 0..8 (0 = auto)");
  if (c->attend_layers < 0) return bad("attend_layers must be >= 0 (0 = auto)");
  if (c->exact_scan < 0 || c->exact_scan > 1) return bad("exact_scan must be 0 or 1");
  if (c->slow_tier_device < -1) return bad("slow_tier_device must be -1 (pinned host) or a device index");
  if (c->dtype != NOSA_DTYPE_BF16 && c->dtype != NOSA_DTYPE_FP32) return bad("dtype must be bf16 or fp32");
  if (c->variant < 0 || c->variant > 2) return bad("variant must be ed-dma, s-dma or dma");
  if (c->residency != NOSA_RESIDENCY_PER_SEQUENCE && c->residency != NOSA_RESIDENCY_SHARED)
    return bad("residency must be per-sequence or shared");
  // the shared-pool victim key packs (last_required << 32 | batch << 16 | block)
  if (c->residency == NOSA_RESIDENCY_SHARED &&
      (c->batch >= 65536 || (c->max_tokens + c->n_b - 1) / c->n_b >= 65536))
    return bad("shared residency needs batch < 65536 and fewer than 65536 blocks per head");
  if (c->n_head / c->n_kv_head > 16) return bad("group size n_head/n_kv_head must be <= 16");
  if (!nosa::attend_supported(c->n_b, c->d_head, c->dtype))
    return bad("unsupported (n_b=%d, d_head=%d, dtype=%d): n_b in {16,32,64,128}, d_head in {64,128}",
               c->n_b, c->d_head, c->dtype);
  return NOSA_OK;
}

extern "C" int nosa_config_budgets(const NosaConfig* c, int32_t* bq, int32_t* be, int32_t* bt) {
  int q, e, t;
  budgets(*c, &q, &e, &t);
  if (bq) *bq = q;
  if (be) *be = e;
  if (bt) *bt = t;
  return NOSA_OK;
}

template <typename T>
static int dalloc(NosaCtx* ctx, T** p, size_t count) {
  const size_t bytes = std::max<size_t>(count * sizeof(T), 16);
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), bytes);
  if (e != cudaSuccess)
    return fail(ctx, NOSA_ERR_CUDA, "cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
  cudaMemset(*p, 0, bytes);
  ctx->dev_allocs.push_back(*p);
  ctx->dev_bytes += bytes;
  return NOSA_OK;
}

static void release(NosaCtx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  delete ctx->pack;
  for (auto* evs : {&ctx->hp_ev_dma, &ctx->hp_ev_sc})
    for (auto e : *evs) cudaEventDestroy(e);
  if (ctx->hp_host) cudaFreeHost(ctx->hp_host);
  if (ctx->hp_dev) cudaFree(ctx->hp_dev);
  if (ctx->hp_xdst) cudaFree(ctx->hp_xdst);
  if (ctx->scatter_stream) cudaStreamDestroy(ctx->scatter_stream);
  if (ctx->smg_stream) cudaStreamDestroy(ctx->smg_stream);
  for (auto e : ctx->ev_smg) cudaEventDestroy(e);
  for (cudaGraphExec_t x : {ctx->graph_exec, ctx->graph_exec_timed, ctx->graph_exec_host})
    if (x) cudaGraphExecDestroy(x);
  for (cudaGraph_t x : {ctx->graph, ctx->graph_timed, ctx->graph_host})
    if (x) cudaGraphDestroy(x);
  for (auto* evs : {&ctx->ev_plan, &ctx->ev_gather, &ctx->ev_att, &ctx->ev_fin, &ctx->ev_in})
    for (auto e : *evs) cudaEventDestroy(e);
  for (cudaEvent_t e : {ctx->ev_fork, ctx->ev_d2h})
    if (e) cudaEventDestroy(e);
  for (cudaStream_t s : {ctx->sel_stream, ctx->copy_stream, ctx->capture_stream, ctx->att_stream, ctx->att_stream2, ctx->fin_stream,
                         ctx->meta_stream, ctx->d2h_stream, ctx->in_stream})
    if (s) cudaStreamDestroy(s);
  if (ctx->h_list) cudaFreeHost(ctx->h_list);
  if (ctx->h_cnt) cudaFreeHost(ctx->h_cnt);
  for (void* p : {(void*)ctx->h_xsrc, (void*)ctx->h_xdst, (void*)ctx->h_xcnt})
    if (p) cudaFreeHost(p);
  for (auto* pool : {&ctx->timing, &ctx->cap_events})
    for (auto& t : *pool) {
      cudaEventDestroy(t.a);
      cudaEventDestroy(t.b);
    }
  for (void* p : ctx->dev_allocs) cudaFree(p);
  if (ctx->staging) cudaFree(ctx->staging);
  if (ctx->io_buf) cudaFree(ctx->io_buf);
  if (ctx->hid_buf) cudaFree(ctx->hid_buf);
  if (ctx->dv.ktime) cudaFree(ctx->dv.ktime);
  if (ctx->dv.sel_prof) cudaFree(ctx->dv.sel_prof);
  if (ctx->proj_wbuf) cudaFree(ctx->proj_wbuf);
  if (ctx->host_mirror && ctx->mirror_device >= 0) {
    cudaSetDevice(ctx->mirror_device);
    cudaFree(ctx->host_mirror);
    cudaSetDevice(ctx->device);
  } else if (ctx->host_mirror) {
    if (ctx->host_registered) {
      cudaHostUnregister(ctx->host_mirror);
      munmap(ctx->host_mirror, ctx->host_bytes);
    } else {
      cudaFreeHost(ctx->host_mirror);
    }
  }
  delete ctx;
}

extern "C" int nosa_ctx_create(const NosaConfig* cfg, int device, NosaCtx** out) {
  char msg[512];
  if (!out) return fail(nullptr, NOSA_ERR_VALUE, "out is NULL");
  *out = nullptr;
  if (nosa_config_validate(cfg, msg, sizeof(msg)) != NOSA_OK) return fail(nullptr, NOSA_ERR_VALUE, "%s", msg);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(nullptr, NOSA_ERR_CUDA, "no CUDA device visible (this path has no CPU fallback)");
  if (device < 0 || device >= ndev) return fail(nullptr, NOSA_ERR_VALUE, "device %d out of range", device);
  cudaSetDevice(device);
  cudaDeviceProp prop{};
  cudaGetDeviceProperties(&prop, device);
  if (prop.major < 10)
    return fail(nullptr, NOSA_ERR_CUDA, "device %d is sm_%d%d; this library is built for sm_100a", device,
                prop.major, prop.minor);

  NosaCtx* ctx = new NosaCtx();
  ctx->cfg = *cfg;
  ctx->device = device;
  ctx->num_sms = prop.multiProcessorCount;
  if (const char* g = getenv("NOSA_GATHER_CTAS")) ctx->gather_grid = ctx->tma_gather_grid = std::max(1, atoi(g));
  const NosaConfig& c = *cfg;
  Dev& dv = ctx->dv;
  dv.B = c.batch;
  dv.H = c.n_kv_head;
  dv.Hq = c.n_head;
  dv.G = c.n_head / c.n_kv_head;
  dv.D = c.d_head;
  dv.n_b = c.n_b;
  dv.n_s = c.n_s;
  dv.n_w = c.n_w;
  dv.n_sink = c.n_s / c.n_b;
  budgets(c, &dv.m_q, &dv.m_e, &dv.m_topk);
  dv.MQ = std::max(dv.m_topk, 1);
  dv.ME = std::max(dv.m_e, 1);
  dv.L = c.layers;
  dv.C = c.fast_slots;
  dv.NB = (c.max_tokens + c.n_b - 1) / c.n_b;
  dv.n_ev = c.n_head;
  dv.dtype = c.dtype;
  dv.variant = c.variant;
  dv.shared = c.residency == NOSA_RESIDENCY_SHARED;
  dv.screen = (c.exact_scan == 0 && (c.d_head == 128 || c.d_head == 64) && !getenv("NOSA_EXACT_SCAN")) ? 1 : 0;
  dv.elem = c.dtype == NOSA_DTYPE_BF16 ? 2 : 4;
  dv.bpb = 2LL * c.n_b * c.d_head * dv.elem;
  // blocks over 32 KiB (fp32 storage): 12 gather CTAs with two blocks each in flight
  // (cfg 3 fp32: 48.2 GB/s vs 39.8 with 8 CTAs of one block; tools/r2bb.sh)
  if (dv.bpb > 32768 && !getenv("NOSA_GATHER_CTAS")) ctx->gather_grid = 12;
  // split-K chunk: the largest of 8, 4, 2, 1 blocks that still gives every SM two work
  // items per layer (measured: smaller chunks cost more in per-chunk overhead than they win in
  // balance once there are a few waves) (B*H*|R| blocks, |R| ~ fixed + top-k), so a small batch does not leave
  // SMs idle in the last wave; a caller that needs bit-identical outputs across batch sizes
  // (e.g. strong scaling over GPUs) pins it with NosaConfig.attend_chunk
  if (c.attend_chunk > 0) {
    dv.chunk = std::min(c.attend_chunk, nosa::kChunk);
  } else {
    const long long r_est = (long long)dv.n_sink + c.n_w / c.n_b + 1 + dv.m_topk;
    const long long blocks = (long long)dv.B * dv.H * std::min<long long>(r_est, dv.C);
    dv.chunk = nosa::kChunk;
    while (dv.chunk > 1 && blocks / dv.chunk < 2LL * ctx->num_sms) dv.chunk >>= 1;
  }
  if (const char* e = getenv("NOSA_CHUNK")) dv.chunk = std::max(1, std::min(atoi(e), nosa::kChunk));
  dv.max_chunks = (dv.C + dv.chunk - 1) / dv.chunk;
  // layers per attention launch (pipelined schedule): when every block of a sequence fits in
  // HBM the step is HBM-bound and per-launch ramp-up/drain is the loss, so 8 layers share one
  // persistent launch (measured on cfg 2: 1 / 4 / 6 / 7 / 8 / 10 / 14 layers per launch =
  // 37.0K / 44.7K / 45.7K / 45.4K / 46.3-46.5K / 46.5K / 45.7K tok/s); with offloaded blocks each
  // layer's attention waits only for its own miss transfer.  fp32 runs one layer per launch.
  // With offloaded blocks the step is bound by the miss transfers, one layer after another; the
  // attention of a batch of layers starts once the batch's last transfer lands, so the plan ramps
  // 1, 4, 4, ..., 2, 1: the first and last layers' attention follow their own transfer at once
  // (the step's head and tail), the middle layers share launches, which amortises the launch and
  // dependency latency of each persistent launch (measured on cfg 3: 1 / 2 / 4 layers per launch
  // = 0.74 / 0.89 / 0.97 of HBM bandwidth per launch by CUDA events; uniform 2 and 4 lengthen the
  // step's tail by 1 and 3 attention layers).
  std::vector<int>& plan = ctx->att_plan;
  plan.clear();
  const bool uniform_req = c.attend_layers > 0 || getenv("NOSA_ATTEND_LAYERS");
  if (c.dtype != NOSA_DTYPE_BF16 && nosa::attend_f32_per_layer()) {
    plan.assign(dv.L, 1);
  } else if (const char* e = getenv("NOSA_ATTEND_PLAN")) {  // experiments: "a,b,c,..." (summing to L)
    int sum = 0;
    for (const char* x = e; *x;) {
      const int v = std::max(1, atoi(x));
      plan.push_back(std::min(v, dv.L - sum));
      sum += plan.back();
      while (*x && *x != ',') ++x;
      if (*x == ',') ++x;
      if (sum >= dv.L) break;
    }
    if (sum < dv.L) plan.push_back(dv.L - sum);
  } else if (uniform_req || dv.C >= dv.NB) {
    int nl = c.attend_layers > 0 ? c.attend_layers : (dv.C >= dv.NB ? 8 : 1);
    if (const char* e = getenv("NOSA_ATTEND_LAYERS")) nl = std::max(1, atoi(e));
    nl = std::min(nl, dv.L);
    for (int l = 0; l < dv.L; l += nl) plan.push_back(std::min(nl, dv.L - l));
  } else {
    if (dv.L <= 3) {
      plan.assign(dv.L, 1);
    } else {
      plan.push_back(1);
      int mid = dv.L - 4;
      for (; mid >= 4; mid -= 4) plan.push_back(4);
      if (mid) plan.push_back(mid);
      plan.push_back(2);
      plan.push_back(1);
    }
  }
  ctx->attend_layers = *std::max_element(plan.begin(), plan.end());
  dv.nbuf = 2 * ctx->attend_layers;
  const size_t LBH = (size_t)dv.L * dv.B * dv.H;
  const size_t BH = (size_t)dv.B * dv.H;

  int rc = NOSA_OK;
#define ALLOC(p, n)                                                   \
  if ((rc = dalloc(ctx, &(p), (n))) != NOSA_OK) {                     \
    g_create_error = ctx->err;                                        \
    release(ctx);                                                     \
    return rc;                                                        \
  }
  char* pool = nullptr;
  ALLOC(pool, LBH * dv.C * (size_t)dv.bpb);
  dv.pool = pool;
  ALLOC(dv.kc, LBH * dv.NB * dv.D);
  ALLOC(dv.se, LBH * dv.NB);
  ALLOC(dv.tail_ksum, LBH * dv.D);
  ALLOC(dv.tail_se, LBH);
  ALLOC(dv.rank_e, LBH * dv.NB);
  ALLOC(dv.slot_of, LBH * dv.NB);
  ALLOC(dv.blk_of, LBH * dv.C);
  ALLOC(dv.lastreq, LBH * dv.C);
  ALLOC(dv.fstack, LBH * dv.C);
  ALLOC(dv.ftop, LBH);
  ALLOC(dv.clock, LBH);
  ALLOC(dv.t, LBH);
  ALLOC(dv.t0, LBH);
  ALLOC(dv.stats, LBH * nosa::ST_N);
  ALLOC(dv.req, LBH * dv.C);
  ALLOC(dv.req_slot, LBH * dv.C);
  ALLOC(dv.n_req, LBH);
  ALLOC(dv.sel_q, LBH * dv.MQ);
  ALLOC(dv.n_selq, LBH);
  ALLOC(dv.sel_e, LBH * dv.ME);
  ALLOC(dv.n_sele, LBH);
  ALLOC(dv.s_q, LBH * dv.NB);
  if (dv.screen) {
    ALLOC(dv.kc16, LBH * dv.NB * dv.D);
    ALLOC(dv.kc_err, LBH * dv.NB);
    ALLOC(dv.qsum_buf, LBH * dv.D);
    // the screen scan inside select_plan (fused, default) or as its own kernel ahead of it
    // (NOSA_SPLIT_SCAN=1).  Measured (tools/r2y.sh, two alternations): cfg 2 46.3K vs 45.2K tok/s
    // fused / split, 31 vs 38 us per 8-layer selection group; cfg 3 14.06K vs 14.15K (within
    // run-to-run spread).  Fused, one CTA's scan overlaps another CTA's sort and plan on the SM.
    dv.split_scan = getenv("NOSA_SPLIT_SCAN") ? 1 : 0;
    if (dv.split_scan) {
      ALLOC(dv.scr_lo, LBH * dv.NB);
      ALLOC(dv.scr_up, LBH * dv.NB);
    }
  }
  ALLOC(dv.plan_fetch, LBH * dv.C);
  ALLOC(dv.plan_evict, LBH * dv.C);
  ALLOC(dv.plan_n, LBH * 3);
  ALLOC(dv.cnt, (size_t)dv.L * nosa::kCntStride);
  ALLOC(dv.miss_list, (size_t)dv.L * BH * dv.C);
  ALLOC(dv.part_o, (size_t)dv.nbuf * BH * dv.max_chunks * dv.G * dv.D);
  ALLOC(dv.part_ml, (size_t)dv.nbuf * BH * dv.max_chunks * dv.G);
  ALLOC(dv.newrow, LBH * 2 * dv.D * (size_t)dv.elem);
  ALLOC(dv.w1, (size_t)dv.D * dv.n_ev);
  ALLOC(dv.w2, (size_t)dv.n_ev);
  ALLOC(dv.err, 1);
#undef ALLOC
  // every slot free, every block slow-resident (offload_sim.py:262-266)
  {
    std::vector<int> neg((size_t)std::max<size_t>(LBH * dv.NB, LBH * dv.C), -1);
    cudaMemcpy(dv.slot_of, neg.data(), LBH * dv.NB * sizeof(int), cudaMemcpyHostToDevice);
    cudaMemcpy(dv.blk_of, neg.data(), LBH * dv.C * sizeof(int), cudaMemcpyHostToDevice);
    // per-sequence pools: [C-1 .. 0] per row; shared pools: row (l, b, h) holds entries
    // [b*C, b*C + C) of the (l, h) stack [B*C-1 .. 0] (kv_manager.py:147-150)
    const int n_free = dv.shared ? dv.B * dv.C : dv.C;
    std::vector<int> stack(LBH * dv.C), top(LBH, n_free);
    for (size_t x = 0; x < LBH; ++x) {
      const int b = (int)((x / dv.H) % dv.B);
      for (int i = 0; i < dv.C; ++i) stack[x * dv.C + i] = n_free - 1 - ((dv.shared ? b * dv.C : 0) + i);
    }
    cudaMemcpy(dv.fstack, stack.data(), stack.size() * sizeof(int), cudaMemcpyHostToDevice);
    cudaMemcpy(dv.ftop, top.data(), top.size() * sizeof(int), cudaMemcpyHostToDevice);
  }

  // slow tier: pinned + mapped host mirror, or (slow_tier_device >= 0) a buffer in that GPU's
  // HBM, read over NVLink by peer access; the same device = loopback
  ctx->host_bytes = LBH * dv.NB * (size_t)dv.bpb;
  // cudaHostAlloc by default.  Measured: an mmap(MADV_HUGEPAGE) + cudaHostRegister mirror pins
  // 2.4x faster at setup, but over a few dozen steps the GPU's writes and reads to it stall for
  // milliseconds at random (cfg 3: 8.6 -> 10.5 ms/step, cfg 2 steps from 0.8 to 8 ms), so it is
  // opt-in (NOSA_HOST_ALLOC=register).
  const char* hmode = getenv("NOSA_HOST_ALLOC");
  const bool use_register = hmode && strcmp(hmode, "register") == 0;
  cudaError_t he = cudaErrorMemoryAllocation;
  if (c.slow_tier_device >= 0) {
    const int peer = c.slow_tier_device;
    if (peer != device) {
      int can = 0;
      cudaDeviceCanAccessPeer(&can, device, peer);
      if (!can) {
        fail(ctx, NOSA_ERR_VALUE, "device %d cannot access device %d's memory (no peer path)", device, peer);
        g_create_error = ctx->err;
        release(ctx);
        return NOSA_ERR_VALUE;
      }
      cudaError_t pe = cudaDeviceEnablePeerAccess(peer, 0);
      if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) {
        fail(ctx, NOSA_ERR_CUDA, "enable peer access %d -> %d: %s", device, peer, cudaGetErrorString(pe));
        g_create_error = ctx->err;
        release(ctx);
        return NOSA_ERR_CUDA;
      }
      cudaGetLastError();
      cudaSetDevice(peer);
    }
    he = cudaMalloc(reinterpret_cast<void**>(&ctx->host_mirror), std::max<size_t>(ctx->host_bytes, 16));
    cudaSetDevice(device);
    if (he != cudaSuccess) {
      ctx->host_mirror = nullptr;
      fail(ctx, NOSA_ERR_CUDA, "slow tier of %zu bytes on device %d: %s", ctx->host_bytes, peer, cudaGetErrorString(he));
      g_create_error = ctx->err;
      release(ctx);
      return NOSA_ERR_CUDA;
    }
    ctx->mirror_device = peer;
    // over NVLink the SM mover is bounded by loads in flight, not by a 55 GB/s link: one CTA
    // per SM (measured on the loopback tier: 8 CTAs 117 GB/s, 64 CTAs 258 GB/s; the copy
    // engine moves 32 KiB device-to-device blocks at 8 GB/s)
    if (!getenv("NOSA_GATHER_CTAS")) ctx->gather_grid = ctx->num_sms;
  } else if (use_register) {
    void* p = mmap(nullptr, ctx->host_bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p != MAP_FAILED) {
      madvise(p, ctx->host_bytes, MADV_HUGEPAGE);
      he = cudaHostRegister(p, ctx->host_bytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
      if (he == cudaSuccess) {
        ctx->host_mirror = static_cast<char*>(p);
        ctx->host_registered = true;
      } else {
        munmap(p, ctx->host_bytes);
      }
    }
  }
  if (!ctx->host_mirror) {
    he = cudaHostAlloc(reinterpret_cast<void**>(&ctx->host_mirror), std::max<size_t>(ctx->host_bytes, 16),
                       cudaHostAllocMapped | cudaHostAllocPortable);
    if (he != cudaSuccess) {
      ctx->host_mirror = nullptr;
      fail(ctx, NOSA_ERR_CUDA, "pinned host mirror of %zu bytes: %s", ctx->host_bytes, cudaGetErrorString(he));
      g_create_error = ctx->err;
      release(ctx);
      return NOSA_ERR_CUDA;
    }
  }
  void* hdev = ctx->host_mirror;
  if (ctx->mirror_device < 0) cudaHostGetDevicePointer(&hdev, ctx->host_mirror, 0);
  dv.host = static_cast<char*>(hdev);

  // Stream priorities (levels below the device's highest; 0 = highest): every stage of the step
  // at the highest level, so the step's kernels go ahead of other work on the device.  Measured
  // on cfg 2/3 (NOSA_PRIO="sel,copy,attend,finalize" overrides): ordering the stages by
  // priority (selection > transfer > attention > merge) moved the step time within run-to-run
  // noise (±5%).
  int prio_low = 0, prio_high = 0;
  cudaDeviceGetStreamPriorityRange(&prio_low, &prio_high);
  int lvl[4] = {0, 0, 0, 0};
  if (const char* e = getenv("NOSA_PRIO")) sscanf(e, "%d,%d,%d,%d", &lvl[0], &lvl[1], &lvl[2], &lvl[3]);
  const bool use_prio = !(getenv("NOSA_NO_STREAM_PRIORITY"));
  auto prio = [&](int k) { return use_prio ? std::min(prio_low, prio_high + std::max(0, k)) : 0; };
  cudaStreamCreateWithPriority(&ctx->sel_stream, cudaStreamNonBlocking, prio(lvl[0]));
  cudaStreamCreateWithPriority(&ctx->copy_stream, cudaStreamNonBlocking, prio(lvl[1]));
  cudaStreamCreateWithPriority(&ctx->att_stream, cudaStreamNonBlocking, prio(lvl[2]));
  cudaStreamCreateWithPriority(&ctx->att_stream2, cudaStreamNonBlocking, prio(lvl[2]));
  ctx->two_att = !getenv("NOSA_ONE_ATT_STREAM");
  ctx->select_per_layer = getenv("NOSA_SELECT_PER_LAYER") != nullptr;
  ctx->stage_with_copies = getenv("NOSA_STAGE_COPIES") != nullptr;
  if (const char* g = getenv("NOSA_STAGE_CTAS")) ctx->stage_grid = std::max(1, atoi(g));
  cudaStreamCreateWithPriority(&ctx->fin_stream, cudaStreamNonBlocking, prio(lvl[3]));
  cudaStreamCreateWithFlags(&ctx->capture_stream, cudaStreamNonBlocking);
  cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming);
  for (auto* evs : {&ctx->ev_plan, &ctx->ev_gather, &ctx->ev_att, &ctx->ev_fin}) {
    evs->resize(dv.L);
    for (int l = 0; l < dv.L; ++l) cudaEventCreateWithFlags(&(*evs)[l], cudaEventDisableTiming);
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    fail(ctx, NOSA_ERR_CUDA, "context init: %s", cudaGetErrorString(e));
    g_create_error = ctx->err;
    release(ctx);
    return NOSA_ERR_CUDA;
  }
  *out = ctx;
  return NOSA_OK;
}

extern "C" void nosa_ctx_destroy(NosaCtx* ctx) { release(ctx); }

extern "C" const char* nosa_last_error(const NosaCtx* ctx) {
  return ctx ? ctx->err.c_str() : g_create_error.c_str();
}

extern "C" int nosa_ctx_memory(const NosaCtx* ctx, int64_t* dev, int64_t* host) {
  if (!ctx) return NOSA_ERR_VALUE;
  if (dev) *dev = (int64_t)ctx->dev_bytes;
  if (host) *host = (int64_t)ctx->host_bytes;
  return NOSA_OK;
}

extern "C" int64_t nosa_launch_count(const NosaCtx* ctx) { return ctx ? ctx->launches.load() : 0; }

extern "C" int nosa_set_eviction_head(NosaCtx* ctx, const double* w1, const double* w2) {
  if (!ctx || !w1 || !w2) return fail(ctx, NOSA_ERR_VALUE, "eviction head weights are NULL");
  cudaSetDevice(ctx->device);
  CUDA_TRY(ctx, cudaMemcpy(ctx->dv.w1, w1, sizeof(double) * ctx->dv.D * ctx->dv.n_ev, cudaMemcpyHostToDevice));
  CUDA_TRY(ctx, cudaMemcpy(ctx->dv.w2, w2, sizeof(double) * ctx->dv.n_ev, cudaMemcpyHostToDevice));
  ctx->have_evhead = true;
  return NOSA_OK;
}

static inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

static int check_layer(NosaCtx* ctx, int layer) {
  if (!ctx) return NOSA_ERR_VALUE;
  if (layer < 0 || layer >= ctx->dv.L) return fail(ctx, NOSA_ERR_VALUE, "layer %d out of range [0, %d)", layer, ctx->dv.L);
  return NOSA_OK;
}

extern "C" int nosa_prefill(NosaCtx* ctx, int layer, int seq_begin, int seq_count, const void* k,
                            const void* v, int t, void* stream) {
  int rc = check_layer(ctx, layer);
  if (rc) return rc;
  const Dev& dv = ctx->dv;
  if (!ctx->have_evhead) return fail(ctx, NOSA_ERR_STATE, "set the eviction head before prefill");
  if (seq_begin < 0 || seq_count <= 0 || seq_begin + seq_count > dv.B)
    return fail(ctx, NOSA_ERR_VALUE, "sequence range [%d, %d) outside batch %d", seq_begin, seq_begin + seq_count, dv.B);
  if (t < 0 || t > ctx->cfg.max_tokens)
    return fail(ctx, NOSA_ERR_VALUE, "head cache capacity exhausted: prefill of %d tokens > max_tokens %d", t,
                ctx->cfg.max_tokens);
  if (t > 0 && (!k || !v)) return fail(ctx, NOSA_ERR_VALUE, "k/v are NULL");
  if (dv.shared && (seq_begin != 0 || seq_count != dv.B))
    return fail(ctx, NOSA_ERR_VALUE, "a shared-pool context prefills the whole batch of a layer at once");
  cudaSetDevice(ctx->device);
  const size_t need = (size_t)seq_count * dv.H * dv.NB * (size_t)dv.bpb;
  if (need > ctx->staging_bytes) {
    cudaStreamSynchronize(S(stream));
    if (ctx->staging) cudaFree(ctx->staging);
    ctx->staging = nullptr;
    CUDA_TRY(ctx, cudaMalloc(&ctx->staging, need));
    ctx->staging_bytes = need;
  }
  CUDA_TRY(ctx, nosa::launch_prefill(dv, layer, seq_begin, seq_count, k, v, t, ctx->staging, S(stream)));
  ctx->launches += 3;
  ctx->prefilled_resident.resize((size_t)dv.L * dv.B, 0);
  for (int b = seq_begin; b < seq_begin + seq_count; ++b) ctx->prefilled_resident[(size_t)layer * dv.B + b] = 0;
  const size_t lbh0 = ((size_t)layer * dv.B + seq_begin) * dv.H;
  CUDA_TRY(ctx, cudaMemcpyAsync(ctx->host_mirror + lbh0 * dv.NB * (size_t)dv.bpb, ctx->staging, need,
                                cudaMemcpyDefault, S(stream)));  // host, or a peer GPU's HBM
  return NOSA_OK;
}

extern "C" int nosa_prefill_resident(NosaCtx* ctx, int layer, int seq_begin, int seq_count, const void* k,
                                     const void* v, int t, void* stream) {
  if (ctx && ctx->dv.shared) return fail(ctx, NOSA_ERR_VALUE, "resident prefill needs per-sequence residency");
  int rc = nosa_prefill(ctx, layer, seq_begin, seq_count, k, v, t, stream);
  if (rc) return rc;
  const Dev& dv = ctx->dv;
  const int nblk = (t + dv.n_b - 1) / dv.n_b;
  if (nblk > dv.C)
    return fail(ctx, NOSA_ERR_CAPACITY, "resident prefill of %d blocks needs fast_slots >= %d (have %d)", nblk, nblk,
                dv.C);
  if (nblk == 0) return NOSA_OK;
  // the swizzled blocks are still in the staging buffer: copy them to slots [0, nblk) of every
  // (sequence, head) and map block i -> slot i (allocate(FAST, ...) in block order)
  const size_t lbh0 = ((size_t)layer * dv.B + seq_begin) * dv.H;
  CUDA_TRY(ctx, cudaMemcpy2DAsync(dv.pool + lbh0 * dv.C * (size_t)dv.bpb, (size_t)dv.C * dv.bpb, ctx->staging,
                                  (size_t)dv.NB * dv.bpb, (size_t)nblk * dv.bpb, (size_t)seq_count * dv.H,
                                  cudaMemcpyDeviceToDevice, S(stream)));
  CUDA_TRY(ctx, nosa::launch_make_resident(dv, layer, seq_begin, seq_count, nblk, S(stream)));
  ctx->launches += 1;
  for (int b = seq_begin; b < seq_begin + seq_count; ++b) ctx->prefilled_resident[(size_t)layer * dv.B + b] = 1;
  return NOSA_OK;
}

extern "C" int nosa_start_run(NosaCtx* ctx, int seq_begin, int seq_count, void* stream) {
  if (!ctx) return NOSA_ERR_VALUE;
  if (seq_begin < 0 || seq_count <= 0 || seq_begin + seq_count > ctx->dv.B)
    return fail(ctx, NOSA_ERR_VALUE, "sequence range outside batch");
  cudaSetDevice(ctx->device);
  // All-resident run: every (layer, sequence) prefilled into HBM and room for every block the
  // run can create (fast_slots >= blocks of max_tokens), so nothing is ever evicted and the only
  // misses are newborn blocks, which the planner rebuilds itself (no gather launch per layer).
  {
    Dev& dv = ctx->dv;
    ctx->prefilled_resident.resize((size_t)dv.L * dv.B, 0);
    bool all = !dv.shared && dv.C >= dv.NB && !getenv("NOSA_GATHER_ALWAYS");
    for (char r : ctx->prefilled_resident) all = all && r;
    dv.born_local = all ? 1 : 0;
  }
  CUDA_TRY(ctx, nosa::launch_start_run(ctx->dv, seq_begin, seq_count, S(stream)));
  ctx->launches += 1;
  if (ctx->dv.screen) {
    CUDA_TRY(ctx, nosa::launch_screen_build(ctx->dv, seq_begin, seq_count, S(stream)));
    ctx->launches += 1;
  }
  return NOSA_OK;
}

// kernels one selection launch issues: the screen scan (split, Dev::split_scan) + select_plan
static int sel_kernels(const Dev& dv) { return dv.screen && dv.split_scan ? 2 : 1; }

// K1+K2 for one layer: fused per-(sequence, head) select+plan, or select then the ordered
// shared-pool planner (NOSA_RESIDENCY_SHARED)
static cudaError_t plan_layer(NosaCtx* ctx, int layer, const void* q, int selector, cudaStream_t st,
                              int export_mode = 0) {
  const Dev& dv = ctx->dv;
  if (!dv.shared) {
    Dev dx = dv;
    dx.x_on = export_mode != 0;
    if (export_mode == 2) dx.x_dst = ctx->hp_xdst;  // host-pack: slot addresses stay on the device
    dx.x_split = export_mode == 2 ? ctx->hp_split : 1024;
    return nosa::launch_select_plan(dx, layer, q, selector, 1, nullptr, nullptr, st);
  }
  cudaError_t e = nosa::launch_select_plan(dv, layer, q, selector, 0, nullptr, nullptr, st);
  if (e != cudaSuccess) return e;
  return nosa::launch_plan_shared(dv, layer, nullptr, nullptr, st);
}

extern "C" int nosa_select_plan(NosaCtx* ctx, int layer, const void* q, int selector, void* stream) {
  int rc = check_layer(ctx, layer);
  if (rc) return rc;
  if (selector != 0 && selector != 1) return fail(ctx, NOSA_ERR_VALUE, "selector must be nosa or infllmv2");
  cudaSetDevice(ctx->device);
  CUDA_TRY(ctx, cudaMemsetAsync(ctx->dv.cnt + nosa::kCntStride * layer, 0, nosa::kCntStride * sizeof(int), S(stream)));
  CUDA_TRY(ctx, plan_layer(ctx, layer, q, selector, S(stream)));
  ctx->launches += sel_kernels(ctx->dv) + (ctx->dv.shared ? 1 : 0);
  return NOSA_OK;
}

extern "C" int nosa_select(NosaCtx* ctx, int layer, const void* q, int selector, void* stream) {
  int rc = check_layer(ctx, layer);
  if (rc) return rc;
  if (selector != 0 && selector != 1) return fail(ctx, NOSA_ERR_VALUE, "selector must be nosa or infllmv2");
  cudaSetDevice(ctx->device);
  CUDA_TRY(ctx, nosa::launch_select_plan(ctx->dv, layer, q, selector, 0, nullptr, nullptr, S(stream)));
  ctx->launches += sel_kernels(ctx->dv);
  return NOSA_OK;
}

extern "C" int nosa_cache_plan(NosaCtx* ctx, int layer, const int32_t* req, const int32_t* n_req, void* stream) {
  int rc = check_layer(ctx, layer);
  if (rc) return rc;
  if (!req || !n_req) return fail(ctx, NOSA_ERR_VALUE, "required sets are NULL");
  cudaSetDevice(ctx->device);
  CUDA_TRY(ctx, cudaMemsetAsync(ctx->dv.cnt + nosa::kCntStride * layer, 0, nosa::kCntStride * sizeof(int), S(stream)));
  if (ctx->dv.shared)
    CUDA_TRY(ctx, nosa::launch_plan_shared(ctx->dv, layer, req, n_req, S(stream)));
  else
    CUDA_TRY(ctx, nosa::launch_select_plan(ctx->dv, layer, nullptr, 0, 2, req, n_req, S(stream)));
  ctx->launches += 1;
  return NOSA_OK;
}

// Copy-engine mover: once the layer's plan (recorded as `plan_done`) has executed, the host
// reads the miss list back through pinned memory and submits one cudaMemcpyAsync per 32 KiB
// block on `copy_st`.  Costs one host wait per layer and one API call per block (host-bound at
// ~2 us a call: an experiment path, the device movers are the default).
static int gather_memcpy(NosaCtx* ctx, int layer, cudaEvent_t plan_done, cudaStream_t copy_st, bool timed) {
  const Dev& dv = ctx->dv;
  if (!ctx->h_list) {
    const size_t cap = (size_t)dv.B * dv.H * dv.C;
    CUDA_TRY(ctx, cudaHostAlloc(reinterpret_cast<void**>(&ctx->h_list), cap * sizeof(int4), cudaHostAllocDefault));
    CUDA_TRY(ctx, cudaHostAlloc(reinterpret_cast<void**>(&ctx->h_cnt), 16, cudaHostAllocDefault));
    CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->meta_stream, cudaStreamNonBlocking));
  }
  CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->meta_stream, plan_done, 0));
  CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_cnt, dv.cnt + nosa::kCntStride * layer, sizeof(int), cudaMemcpyDeviceToHost, ctx->meta_stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->meta_stream));
  const int n = ctx->h_cnt[0];
  if (n == 0) return NOSA_OK;
  CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_list, dv.miss_list + (size_t)layer * dv.B * dv.H * dv.C, n * sizeof(int4),
                                cudaMemcpyDeviceToHost, ctx->meta_stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->meta_stream));
  ctx->b_dst.resize(n);
  ctx->b_src.resize(n);
  int nc = 0, n_born = 0;
  for (int i = 0; i < n; ++i) {
    const int4 m = ctx->h_list[i];
    if (m.w) {  // born by the last append: rebuilt on the device from the stash, not copied
      ++n_born;
      continue;
    }
    ctx->b_src[nc] = ctx->host_mirror + ((size_t)m.x * dv.NB + m.y) * dv.bpb;
    ctx->b_dst[nc] = dv.pool + ((size_t)m.x * dv.C + m.z) * dv.bpb;
    ++nc;
  }
  TimeScope ts(ctx, copy_st, 1, timed);
  if (n_born) {
    CUDA_TRY(ctx, nosa::launch_born(dv, layer, copy_st, std::min(n_born, ctx->num_sms)));
    ctx->memcpy_born_launches += 1;
  }
  if (nc == 0) return NOSA_OK;
  for (int i = 0; i < nc; ++i)
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->b_dst[i], ctx->b_src[i], (size_t)dv.bpb, cudaMemcpyDefault, copy_st));
  return NOSA_OK;
}

// The mapped pinned host arrays the planner writes each layer's copy list into (Dev::x_*).
static int ensure_export(NosaCtx* ctx) {
  if (ctx->h_xsrc) return NOSA_OK;
  Dev& dv = ctx->dv;
  const size_t cap = (size_t)dv.B * dv.H * dv.C;
  CUDA_TRY(ctx, cudaHostAlloc(reinterpret_cast<void**>(&ctx->h_xsrc), dv.L * cap * sizeof(void*), cudaHostAllocMapped));
  CUDA_TRY(ctx, cudaHostAlloc(reinterpret_cast<void**>(&ctx->h_xdst), dv.L * cap * sizeof(void*), cudaHostAllocMapped));
  CUDA_TRY(ctx, cudaHostAlloc(reinterpret_cast<void**>(&ctx->h_xcnt), 2 * dv.L * sizeof(int), cudaHostAllocMapped));
  CUDA_TRY(ctx, cudaHostGetDevicePointer(reinterpret_cast<void**>(&dv.x_src), ctx->h_xsrc, 0));
  CUDA_TRY(ctx, cudaHostGetDevicePointer(reinterpret_cast<void**>(&dv.x_dst), ctx->h_xdst, 0));
  CUDA_TRY(ctx, cudaHostGetDevicePointer(reinterpret_cast<void**>(&dv.x_cnt), ctx->h_xcnt, 0));
  dv.x_src_base = ctx->host_mirror;  // the address the copy engine reads (host or peer HBM)
  return NOSA_OK;
}

// Copy-engine mover inside a step: the layer's planner already wrote the copy list and its
// counts into mapped host memory (select_plan_kernel with Dev::x_on), so once the plan has
// executed (an event query: no device round trip, no copy) the host submits the list, one
// cudaMemcpyAsync per block.  Blocks born by the last append are rebuilt on the device.
static int gather_exported(NosaCtx* ctx, int layer, cudaStream_t copy_st, bool timed) {
  const Dev& dv = ctx->dv;
  cudaError_t e;
  while ((e = cudaEventQuery(ctx->ev_plan[layer])) == cudaErrorNotReady) {
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
  }
  CUDA_TRY(ctx, e);
  const volatile int* xc = ctx->h_xcnt;
  const int n = xc[2 * layer], n_born = xc[2 * layer + 1];
  TimeScope ts(ctx, copy_st, 1, timed);
  if (n_born) {
    CUDA_TRY(ctx, nosa::launch_born(dv, layer, copy_st, std::min(n_born, ctx->num_sms)));
    ctx->memcpy_born_launches += 1;
  }
  if (n == 0) return NOSA_OK;
  const size_t cap = (size_t)dv.B * dv.H * dv.C;
  void** dst = ctx->h_xdst + layer * cap;
  void** src = ctx->h_xsrc + layer * cap;
  for (int i = 0; i < n; ++i)
    CUDA_TRY(ctx, cudaMemcpyAsync(dst[i], src[i], (size_t)dv.bpb, cudaMemcpyDefault, copy_st));
  return NOSA_OK;
}

// Host-pack mover: the planner exported the layer's copy list (host source addresses) and the
// slot address of every entry (device memory, hp_xdst).  Host threads pack the scattered 32 KiB
// blocks into pinned staging chunks; each chunk crosses PCIe as ONE large DMA on the copy engine
// (the link's full rate, no SM loads in flight next to the attention), and a scatter kernel on
// its own stream moves it from the device ring into the slots.  Packing chunk c+1 overlaps the
// DMA of chunk c.  The layer's gather-done event is recorded after its last scatter.
static int ensure_hostpack(NosaCtx* ctx) {
  if (ctx->pack) return NOSA_OK;
  Dev& dv = ctx->dv;
  if (const char* e = getenv("NOSA_PACK_CHUNK")) ctx->pack_chunk = std::max(1, atoi(e));
  if (const char* e = getenv("NOSA_PACK_SLOTS")) ctx->pack_slots = std::max(2, atoi(e));
  int nthreads = 8;
  if (const char* e = getenv("NOSA_PACK_THREADS")) nthreads = std::max(0, atoi(e));
  const size_t ring = (size_t)ctx->pack_slots * ctx->pack_chunk * dv.bpb;
  CUDA_TRY(ctx, cudaHostAlloc(reinterpret_cast<void**>(&ctx->hp_host), ring, cudaHostAllocDefault));
  memset(ctx->hp_host, 0, ring);
  CUDA_TRY(ctx, cudaMalloc(reinterpret_cast<void**>(&ctx->hp_dev), ring));
  const size_t cap = (size_t)dv.B * dv.H * dv.C;
  CUDA_TRY(ctx, cudaMalloc(reinterpret_cast<void**>(&ctx->hp_xdst), dv.L * cap * sizeof(void*)));
  ctx->hp_ev_dma.resize(ctx->pack_slots);
  ctx->hp_ev_sc.resize(ctx->pack_slots);
  for (int i = 0; i < ctx->pack_slots; ++i) {
    CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->hp_ev_dma[i], cudaEventDisableTiming));
    CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->hp_ev_sc[i], cudaEventDisableTiming));
  }
  ctx->hp_used.assign(ctx->pack_slots, 0);
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  CUDA_TRY(ctx, cudaStreamCreateWithPriority(&ctx->scatter_stream, cudaStreamNonBlocking, hi));
  CUDA_TRY(ctx, cudaStreamCreateWithPriority(&ctx->smg_stream, cudaStreamNonBlocking, hi));
  ctx->ev_smg.resize(dv.L);
  for (auto& e : ctx->ev_smg) CUDA_TRY(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  ctx->pack = new PackPool();
  ctx->pack->start(nthreads);
  return NOSA_OK;
}

static int gather_hostpack(NosaCtx* ctx, int layer, cudaStream_t copy_st, bool timed, bool hybrid) {
  const Dev& dv = ctx->dv;
  cudaError_t e;
  while ((e = cudaEventQuery(ctx->ev_plan[layer])) == cudaErrorNotReady) cpu_relax();
  CUDA_TRY(ctx, e);
  const volatile int* xc = ctx->h_xcnt;
  const int n = xc[2 * layer], n_born = xc[2 * layer + 1];
  cudaStream_t sc = ctx->scatter_stream;
  CUDA_TRY(ctx, cudaStreamWaitEvent(sc, ctx->ev_plan[layer], 0));
  if (n_born && !hybrid) {  // (hybrid: the SM gather rebuilds the born blocks)
    CUDA_TRY(ctx, nosa::launch_born(dv, layer, sc, std::min(n_born, ctx->num_sms)));
    ctx->memcpy_born_launches += 1;
  }
  const size_t cap = (size_t)dv.B * dv.H * dv.C;
  char* const* src = reinterpret_cast<char* const*>(ctx->h_xsrc + layer * cap);
  void* const* dst = ctx->hp_xdst + layer * cap;
  {
    TimeScope ts(ctx, copy_st, 1, timed);
    for (int c0 = 0; c0 < n; c0 += ctx->pack_chunk) {
      const int cnt = std::min(ctx->pack_chunk, n - c0);
      const int slot = ctx->hp_next;
      ctx->hp_next = (ctx->hp_next + 1) % ctx->pack_slots;
      char* hbuf = ctx->hp_host + (size_t)slot * ctx->pack_chunk * dv.bpb;
      char* dbuf = ctx->hp_dev + (size_t)slot * ctx->pack_chunk * dv.bpb;
      if (ctx->hp_used[slot]) {  // the host slot is free once its previous DMA has read it
        while ((e = cudaEventQuery(ctx->hp_ev_dma[slot])) == cudaErrorNotReady) cpu_relax();
        CUDA_TRY(ctx, e);
        CUDA_TRY(ctx, cudaStreamWaitEvent(copy_st, ctx->hp_ev_sc[slot], 0));  // device slot: scattered
      }
      ctx->pack->run(src + c0, hbuf, cnt, (size_t)dv.bpb);
      CUDA_TRY(ctx, cudaMemcpyAsync(dbuf, hbuf, (size_t)cnt * dv.bpb, cudaMemcpyHostToDevice, copy_st));
      CUDA_TRY(ctx, cudaEventRecord(ctx->hp_ev_dma[slot], copy_st));
      CUDA_TRY(ctx, cudaStreamWaitEvent(sc, ctx->hp_ev_dma[slot], 0));
      CUDA_TRY(ctx, nosa::launch_scatter(dbuf, dst + c0, cnt, dv.bpb, sc));
      CUDA_TRY(ctx, cudaEventRecord(ctx->hp_ev_sc[slot], sc));
      ctx->hp_used[slot] = 1;
      ctx->memcpy_born_launches += 1;  // (counted with the mover's kernels)
    }
  }
  CUDA_TRY(ctx, cudaEventRecord(ctx->ev_gather[layer], sc));
  return NOSA_OK;
}

extern "C" int nosa_gather(NosaCtx* ctx, int layer, int mode, void* stream) {
  int rc = check_layer(ctx, layer);
  if (rc) return rc;
  cudaSetDevice(ctx->device);
  if (mode == NOSA_GATHER_MEMCPY) {
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev_plan[layer], S(stream)));
    return gather_memcpy(ctx, layer, ctx->ev_plan[layer], S(stream), false);
  }
  if (mode != NOSA_GATHER_UVA && mode != NOSA_GATHER_TMA)
    return fail(ctx, NOSA_ERR_VALUE, "unknown gather mode %d", mode);
  const bool tma = mode == NOSA_GATHER_TMA;
  CUDA_TRY(ctx, nosa::launch_gather(ctx->dv, layer, S(stream), tma ? ctx->tma_gather_grid : ctx->gather_grid, tma));
  ctx->launches += 1;
  return NOSA_OK;
}

extern "C" int nosa_attend(NosaCtx* ctx, int layer, const void* q, const void* k_new, const void* v_new, float* out,
                           void* stream) {
  int rc = check_layer(ctx, layer);
  if (rc) return rc;
  if (!q || !k_new || !v_new || !out) return fail(ctx, NOSA_ERR_VALUE, "attend: NULL tensor");
  cudaSetDevice(ctx->device);
  CUDA_TRY(ctx, nosa::launch_attend(ctx->dv, layer, 1, q, k_new, v_new, out, S(stream), ctx->num_sms));
  CUDA_TRY(ctx, nosa::launch_finalize(ctx->dv, layer, k_new, v_new, out, S(stream)));
  ctx->launches += 2;
  return NOSA_OK;
}

extern "C" int nosa_timing_enable(NosaCtx* ctx, int max_launches) {
  if (!ctx || max_launches < 0) return NOSA_ERR_VALUE;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  // captured event-record nodes may point into the pool: park them on their placeholders
  // before the pool's events are destroyed
  if (ctx->graph_exec_timed && ctx->nodes_on_pool) {
    for (const auto& en : ctx->ev_nodes)
      CUDA_TRY(ctx, cudaGraphExecEventRecordNodeSetEvent(
                        ctx->graph_exec_timed, en.node, en.end ? ctx->cap_events[en.slot].b : ctx->cap_events[en.slot].a));
    ctx->nodes_on_pool = false;
  }
  for (auto& t : ctx->timing) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  ctx->timing.clear();
  ctx->timing_used = 0;
  for (int i = 0; i < max_launches; ++i) {
    NosaCtx::Timed t{};
    CUDA_TRY(ctx, cudaEventCreate(&t.a));
    CUDA_TRY(ctx, cudaEventCreate(&t.b));
    ctx->timing.push_back(t);
  }
  return NOSA_OK;
}

extern "C" int nosa_timing_read(NosaCtx* ctx, double* total_ms, int64_t* launches) {
  if (!ctx || !total_ms || !launches) return NOSA_ERR_VALUE;
  cudaSetDevice(ctx->device);
  CUDA_TRY(ctx, cudaDeviceSynchronize());
  for (int k = 0; k < 7; ++k) {
    total_ms[k] = 0.0;
    launches[k] = 0;
  }
  for (size_t i = 0; i < ctx->timing_used; ++i) {
    float ms = 0.0f;
    CUDA_TRY(ctx, cudaEventElapsedTime(&ms, ctx->timing[i].a, ctx->timing[i].b));
    total_ms[ctx->timing[i].kind] += ms;
    launches[ctx->timing[i].kind] += 1;
  }
  return NOSA_OK;
}

// `hio` (optional): the step's tensors live in host memory.  `io` then points at the
// context's device staging; layer l's q/k/v are copied in on the copy stream ahead of the miss
// gathers (select(l) waits for its own layer only) and its output is copied back on the d2h
// stream as soon as finalize(l) is done, so the read-back of layer l overlaps layer l+1.
extern "C" int nosa_ktime_enable(NosaCtx* ctx, int on) {
  if (!ctx) return NOSA_ERR_VALUE;
  cudaSetDevice(ctx->device);
  CUDA_TRY(ctx, cudaDeviceSynchronize());
  if (on && !ctx->dv.ktime) {
    CUDA_TRY(ctx, cudaMalloc(reinterpret_cast<void**>(&ctx->dv.ktime), 2 * sizeof(unsigned long long) * ctx->dv.L));
  } else if (!on && ctx->dv.ktime) {
    cudaFree(ctx->dv.ktime);
    ctx->dv.ktime = nullptr;
    return NOSA_OK;
  }
  if (ctx->dv.ktime) {
    std::vector<unsigned long long> init(2 * ctx->dv.L);
    for (int l = 0; l < ctx->dv.L; ++l) init[2 * l] = ~0ull, init[2 * l + 1] = 0ull;
    CUDA_TRY(ctx, cudaMemcpy(ctx->dv.ktime, init.data(), init.size() * 8, cudaMemcpyHostToDevice));
  }
  return NOSA_OK;
}

extern "C" int nosa_ktime_read(NosaCtx* ctx, double* span_us) {
  if (!ctx || !span_us || !ctx->dv.ktime) return NOSA_ERR_VALUE;
  cudaSetDevice(ctx->device);
  CUDA_TRY(ctx, cudaDeviceSynchronize());
  std::vector<unsigned long long> v(2 * ctx->dv.L);
  CUDA_TRY(ctx, cudaMemcpy(v.data(), ctx->dv.ktime, v.size() * 8, cudaMemcpyDeviceToHost));
  for (int l = 0; l < ctx->dv.L; ++l)
    span_us[l] = v[2 * l + 1] > v[2 * l] && v[2 * l] != ~0ull ? (double)(v[2 * l + 1] - v[2 * l]) * 1e-3 : 0.0;
  return nosa_ktime_enable(ctx, 1);  // reset
}

extern "C" int nosa_project_qkv(const void* h, int m, int k, const void* w_t, int n, int nq, int nk, void* q,
                                void* k_out, void* v, int splits, void* stream) {
  if (!h || !w_t || !q || !k_out || !v) return fail(nullptr, NOSA_ERR_VALUE, "project_qkv: NULL argument");
  if (m <= 0 || k <= 0 || n <= 0 || splits <= 0 || splits > 8 || nq < 0 || nk < 0 || nq + nk > n)
    return fail(nullptr, NOSA_ERR_VALUE, "project_qkv: bad shape or splits (1..8)");
  if (n % 128 != 0 || k % (64 * splits) != 0)
    return fail(nullptr, NOSA_ERR_VALUE, "project_qkv: needs N %% 128 == 0 and K %% (64 * splits) == 0 (N=%d K=%d)", n, k);
  if (splits == 1 && (nq % 32 || nk % 32))
    return fail(nullptr, NOSA_ERR_VALUE, "project_qkv: one split needs nq and nk multiples of 32 (nq=%d nk=%d)", nq, nk);
  cudaError_t e = nosa::launch_project(h, w_t, m, n, k, splits, q, k_out, v, nq, nk, S(stream));
  if (e != cudaSuccess) return fail(nullptr, NOSA_ERR_CUDA, "project_qkv: %s", cudaGetErrorString(e));
  return NOSA_OK;
}

extern "C" int nosa_project_f32(const float* h, int m, int k, const float* w, int n, float* out, void* stream) {
  if (!h || !w || !out) return fail(nullptr, NOSA_ERR_VALUE, "project_f32: NULL argument");
  if (m <= 0 || k <= 0 || n <= 0) return fail(nullptr, NOSA_ERR_VALUE, "project_f32: bad shape");
  cudaError_t e = nosa::launch_project_f32(h, w, m, k, n, out, S(stream));
  if (e != cudaSuccess) return fail(nullptr, NOSA_ERR_CUDA, "project_f32: %s", cudaGetErrorString(e));
  return NOSA_OK;
}

extern "C" int nosa_select_profile(NosaCtx* ctx, int on, double* cycles) {
  if (!ctx) return NOSA_ERR_VALUE;
  cudaSetDevice(ctx->device);
  CUDA_TRY(ctx, cudaDeviceSynchronize());
  if (cycles && ctx->dv.sel_prof) {
    long long v[16];
    CUDA_TRY(ctx, cudaMemcpy(v, ctx->dv.sel_prof, sizeof(v), cudaMemcpyDeviceToHost));
    for (int i = 0; i < 16; ++i) cycles[i] = (double)v[i];
  }
  if (on) {
    if (!ctx->dv.sel_prof) CUDA_TRY(ctx, cudaMalloc(reinterpret_cast<void**>(&ctx->dv.sel_prof), 16 * sizeof(long long)));
    CUDA_TRY(ctx, cudaMemset(ctx->dv.sel_prof, 0, 16 * sizeof(long long)));
  } else if (ctx->dv.sel_prof) {
    cudaFree(ctx->dv.sel_prof);
    ctx->dv.sel_prof = nullptr;
  }
  return NOSA_OK;
}

extern "C" int nosa_timing_trace(NosaCtx* ctx, int cap, int32_t* kind, float* start_ms, float* end_ms, int32_t* n) {
  if (!ctx || !n || (cap > 0 && (!kind || !start_ms || !end_ms))) return NOSA_ERR_VALUE;
  cudaSetDevice(ctx->device);
  CUDA_TRY(ctx, cudaDeviceSynchronize());
  const int m = (int)std::min<size_t>(ctx->timing_used, (size_t)std::max(cap, 0));
  for (int i = 0; i < m; ++i) {
    const NosaCtx::Timed& t = ctx->timing[i];
    kind[i] = t.kind;
    CUDA_TRY(ctx, cudaEventElapsedTime(&start_ms[i], ctx->timing[0].a, t.a));
    CUDA_TRY(ctx, cudaEventElapsedTime(&end_ms[i], ctx->timing[0].a, t.b));
  }
  *n = m;
  return NOSA_OK;
}

static int enqueue_step(NosaCtx* ctx, const NosaStepIO* io, cudaStream_t st, bool count,
                        const NosaHostStepIO* hio = nullptr, const void* hidden = nullptr,
                        const void* hidden_host = nullptr) {
  const Dev& dv = ctx->dv;
  const size_t qstride = (size_t)dv.B * dv.Hq * dv.D * dv.elem;
  const size_t kstride = (size_t)dv.B * dv.H * dv.D * dv.elem;
  const size_t ostride = (size_t)dv.B * dv.Hq * dv.D;
  const char* q = static_cast<const char*>(io->q);
  const char* kn = static_cast<const char*>(io->k_new);
  const char* vn = static_cast<const char*>(io->v_new);
  const bool timed = count;  // eager steps only (never inside a graph capture)
  // One stream per stage, forked from the caller's stream `st` and linked per layer by events:
  //   [project(group) ->] select(group) [sel] -> gather(l) [copy] -> attend(batch) [att / att2,
  //   alternating] -> finalize(batch) [fin] [-> D2H of the outputs (host step)]
  // so the selection, miss transfer, attention and merge/append of different layers overlap.
  // An attention batch also waits for the finalize that last used its split-K record buffers
  // (nbuf = 2 x layers per batch: double-buffered batches).
  // Layer-pipelined schedule: the selections are issued first (valid when each layer's query is
  // known up front, as with per-layer query streams).  Layer-serial schedule: select(l) waits
  // for finalize(l-1), as when q_{l+1} is computed from layer l's output.
  const bool serial = io->schedule == 1;
  cudaStream_t cp = ctx->copy_stream, at = ctx->att_stream, fn = ctx->fin_stream, ss = ctx->sel_stream;
  CUDA_TRY(ctx, cudaEventRecord(ctx->ev_fork, st));  // side streams start after the caller's work
  cudaStream_t at2 = ctx->two_att ? ctx->att_stream2 : at;
  for (cudaStream_t s : {ss, cp, at, at2, fn}) CUDA_TRY(ctx, cudaStreamWaitEvent(s, ctx->ev_fork, 0));
  // selection groups: doubling layer ranges (1, 1, 2, 4, 8, ...) in the pipelined schedule,
  // one layer each otherwise (serial schedule, shared-pool planner)
  const bool grouped = !serial && !dv.shared && !ctx->select_per_layer;
  std::vector<std::pair<int, int>>& groups = ctx->groups;
  groups.clear();
  if (grouped) {
    // group sizes (nl = layers of the first attention batch): 1, 1, 2, 4, ... when every layer has its
    // own attention launch (offloaded), nl, 2nl, 4nl, ... when attention is batched
    const int nlb = ctx->att_plan[0];  // the first attention batch waits for the first group only
    if (const char* e = getenv("NOSA_SELECT_PLAN")) {  // experiments: "a,b,..." layers per group
      int l0 = 0;
      for (const char* x = e; *x && l0 < dv.L;) {
        const int n = std::min(std::max(1, atoi(x)), dv.L - l0);
        groups.push_back({l0, n});
        l0 += n;
        while (*x && *x != ',') ++x;
        if (*x == ',') ++x;
      }
      if (l0 < dv.L) groups.push_back({l0, dv.L - l0});
    } else if (nlb > 1) {
      // batched attention (all resident): the first batch's group, then doubling (8, 16, 4 at
      // L = 28): measured 46.7K vs 46.4K tok/s for 8, 8, 12 at cfg 2 (tools/r2ac.sh)
      for (int l0 = 0, n = nlb; l0 < dv.L; l0 += n, n *= 2) groups.push_back({l0, std::min(n, dv.L - l0)});
    } else {
      for (int l0 = 0, n = nlb; l0 < dv.L; l0 += n, n = std::max(nlb, l0)) groups.push_back({l0, std::min(n, dv.L - l0)});
    }
  } else {
    for (int l = 0; l < dv.L; ++l) groups.push_back({l, 1});
  }
  // copy-engine mover: the planner exports each layer's copy list to mapped host memory
  const bool hybrid = io->gather_mode == NOSA_GATHER_HYBRID && !dv.born_local;
  const bool hostpack = (io->gather_mode == NOSA_GATHER_HOSTPACK || io->gather_mode == NOSA_GATHER_HYBRID) &&
                        !dv.born_local;
  if (hostpack && (dv.shared || ctx->capturing || ctx->mirror_device >= 0))
    return fail(ctx, NOSA_ERR_VALUE, "the host-pack mover needs per-sequence residency, a host slow tier and an eager step");
  const bool export_misses = hostpack || (io->gather_mode == NOSA_GATHER_MEMCPY && !dv.shared && !dv.born_local &&
                                          !ctx->capturing && !getenv("NOSA_MEMCPY_READBACK"));
  if (export_misses)
    if (int rc = ensure_export(ctx)) return rc;
  if (hostpack)
    if (int rc = ensure_hostpack(ctx)) return rc;
  const int export_mode = hostpack ? 2 : (export_misses ? 1 : 0);
  Dev dx = dv;  // (ensure_export filled the x_* pointers of ctx->dv)
  dx.x_on = export_misses;
  if (hostpack) {
    ctx->hp_split = 1024;
    if (hybrid) {  // NOSA_HOST_SHARE: the host-packed share of the units (default one half)
      const char* e = getenv("NOSA_HOST_SHARE");
      ctx->hp_split = std::min(1024, std::max(0, (int)lround((e ? atof(e) : 0.5) * 1024.0)));
    }
    dx.x_dst = ctx->hp_xdst;  // slot addresses stay on the device (plan_layer does the same)
  }
  dx.x_split = hostpack ? ctx->hp_split : 1024;
  auto select = [&](int l) -> int {
    if (hio) CUDA_TRY(ctx, cudaStreamWaitEvent(ss, ctx->ev_in[l], 0));
    CUDA_TRY(ctx, cudaMemsetAsync(dv.cnt + nosa::kCntStride * l, 0, nosa::kCntStride * sizeof(int), ss));
    {
      TimeScope ts(ctx, ss, 0, timed);
      CUDA_TRY(ctx, plan_layer(ctx, l, q + l * qstride, io->selector, ss, export_mode));
    }
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev_plan[l], ss));
    return NOSA_OK;
  };
  // Pipelined: the layers' selections are launched in groups of doubling size (1, 1, 2, 4, 8,
  // ...), one grid of (B*H, layers) per group, so layer 0's plan (and its miss transfer) starts
  // at once while the later layers' selections fill the whole GPU in a few launches.
  auto select_group = [&](int l0, int n) -> int {
    if (hio) CUDA_TRY(ctx, cudaStreamWaitEvent(ss, ctx->ev_in[l0 + n - 1], 0));
    CUDA_TRY(ctx, cudaMemsetAsync(dv.cnt + nosa::kCntStride * l0, 0, nosa::kCntStride * n * sizeof(int), ss));
    {
      TimeScope ts(ctx, ss, 0, timed);
      CUDA_TRY(ctx, nosa::launch_select_plan(dx, l0, q + l0 * qstride, io->selector, 1, nullptr, nullptr, ss, n));
    }
    for (int l = l0; l < l0 + n; ++l) CUDA_TRY(ctx, cudaEventRecord(ctx->ev_plan[l], ss));
    return NOSA_OK;
  };
  // Issues groups [next_group, upto): the host inputs of the group (three copies, nosa_decode_
  // step_host), then in the pipelined schedule its selection, so a selection is always enqueued
  // after its inputs' event is recorded in this step (a wait on an earlier step's record would
  // read stale inputs).  Inputs go on their own high-priority stream.  Pinned inputs are staged
  // by a small SM kernel: copy-engine copies would run strictly in order with the miss gathers
  // (measured: the gather of layer 0 then waits for every input copy; interleaving the inputs
  // between the gathers leaves bubbles and ends 7% slower end to end).
  // device-visible aliases of the host inputs when they are pinned (cudaHostAlloc / registered);
  // pageable inputs fall back to cudaMemcpyAsync
  const char* hsrc[3] = {nullptr, nullptr, nullptr};
  const char* hsrc_h = nullptr;  // device alias of pinned host hidden states (hidden host step)
  if (hidden_host && !ctx->stage_with_copies) {
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, hidden_host) == cudaSuccess && pa.type == cudaMemoryTypeHost && pa.devicePointer)
      hsrc_h = static_cast<const char*>(pa.devicePointer);
    else
      cudaGetLastError();
  }
  if (hio && hio->q && !ctx->stage_with_copies) {
    const void* hp[3] = {hio->q, hio->k_new, hio->v_new};
    bool all = true;
    for (int i = 0; i < 3; ++i) {
      cudaPointerAttributes pa{};
      if (cudaPointerGetAttributes(&pa, hp[i]) != cudaSuccess || pa.type != cudaMemoryTypeHost || !pa.devicePointer) {
        cudaGetLastError();
        all = false;
        break;
      }
      hsrc[i] = static_cast<const char*>(pa.devicePointer);
    }
    if (!all) hsrc[0] = hsrc[1] = hsrc[2] = nullptr;
  }
  // hidden-state step: layer l's q | k | v are projected from h[l] on the tensor cores on the
  // selection stream, right before the layer's selection (project_qkv, attention.py:67-90)
  int n_proj = 0;
  auto project = [&](int l0, int n) -> int {
    if (!hidden) return NOSA_OK;
    if (hidden_host) CUDA_TRY(ctx, cudaStreamWaitEvent(ss, ctx->ev_in[l0 + n - 1], 0));  // staged h
    const int N = (dv.Hq + 2 * dv.H) * dv.D, d = ctx->proj_d;
    // One split: a group's layers fill the SMs, and each CTA streams its weight rows over the
    // whole K and stores straight from TMEM (measured on cfg 2 with hidden inputs: 42.1K tok/s
    // vs 38.9K with 4-way cluster split-K).  The same sums as QKVProjection(h, splits=1).
    static const int force_splits = getenv("NOSA_PROJ_SPLITS") ? atoi(getenv("NOSA_PROJ_SPLITS")) : 0;
    const int splits = force_splits > 0 && (d / 64) % force_splits == 0 ? force_splits : 1;
    {  // the group's layers in one launch
      TimeScope ts(ctx, ss, 6, timed);
      CUDA_TRY(ctx, nosa::launch_project(static_cast<const char*>(hidden) + (size_t)l0 * dv.B * d * 2,
                                         ctx->proj_wbuf + (size_t)l0 * N * d * 2, dv.B, N, d, splits,
                                         const_cast<char*>(q) + l0 * qstride, const_cast<char*>(kn) + l0 * kstride,
                                         const_cast<char*>(vn) + l0 * kstride, dv.Hq * dv.D, dv.H * dv.D, ss, n));
      ++n_proj;
    }
    return NOSA_OK;
  };
  size_t next_group = 0;
  auto issue_groups = [&](size_t upto) -> int {
    for (; next_group < std::min(upto, groups.size()); ++next_group) {
      const int l0 = groups[next_group].first, n = groups[next_group].second;
      if (hidden_host) {  // the group's hidden states, host -> the device buffer the projection reads
        cudaStream_t in = ctx->in_stream;
        TimeScope ts(ctx, in, 4, timed);
        const size_t hstride = (size_t)dv.B * ctx->proj_d * 2;
        char* dst = const_cast<char*>(static_cast<const char*>(hidden)) + l0 * hstride;
        if (hsrc_h) {
          const void* src[3] = {hsrc_h + l0 * hstride, nullptr, nullptr};
          void* dsts[3] = {dst, nullptr, nullptr};
          const size_t bytes[3] = {n * hstride, 0, 0};
          CUDA_TRY(ctx, nosa::launch_stage_inputs(src, dsts, bytes, ctx->stage_grid, in));
          if (count) ctx->launches += 1;
        } else {
          CUDA_TRY(ctx, cudaMemcpyAsync(dst, static_cast<const char*>(hidden_host) + l0 * hstride, n * hstride,
                                        cudaMemcpyHostToDevice, in));
        }
        CUDA_TRY(ctx, cudaEventRecord(ctx->ev_in[l0 + n - 1], in));
      } else if (hio && hsrc[0]) {  // mapped pinned inputs: the SMs stage them (zero-copy loads)
        cudaStream_t in = ctx->in_stream;
        TimeScope ts(ctx, in, 4, timed);
        const void* src[3] = {hsrc[0] + l0 * qstride, hsrc[1] + l0 * kstride, hsrc[2] + l0 * kstride};
        void* dst[3] = {const_cast<char*>(q) + l0 * qstride, const_cast<char*>(kn) + l0 * kstride,
                        const_cast<char*>(vn) + l0 * kstride};
        const size_t bytes[3] = {n * qstride, n * kstride, n * kstride};
        CUDA_TRY(ctx, nosa::launch_stage_inputs(src, dst, bytes, ctx->stage_grid, in));
        if (count) ctx->launches += 1;  // (counted apart from step_kernels: capture_host adds one per group)
        CUDA_TRY(ctx, cudaEventRecord(ctx->ev_in[l0 + n - 1], in));
      } else if (hio && hio->q) {
        cudaStream_t in = ctx->in_stream;
        TimeScope ts(ctx, in, 4, timed);
        CUDA_TRY(ctx, cudaMemcpyAsync(const_cast<char*>(q) + l0 * qstride,
                                      static_cast<const char*>(hio->q) + l0 * qstride, n * qstride,
                                      cudaMemcpyHostToDevice, in));
        CUDA_TRY(ctx, cudaMemcpyAsync(const_cast<char*>(kn) + l0 * kstride,
                                      static_cast<const char*>(hio->k_new) + l0 * kstride, n * kstride,
                                      cudaMemcpyHostToDevice, in));
        CUDA_TRY(ctx, cudaMemcpyAsync(const_cast<char*>(vn) + l0 * kstride,
                                      static_cast<const char*>(hio->v_new) + l0 * kstride, n * kstride,
                                      cudaMemcpyHostToDevice, in));
        CUDA_TRY(ctx, cudaEventRecord(ctx->ev_in[l0 + n - 1], in));
      }
      if (!serial) {
        if (int rc = project(l0, n)) return rc;
        if (grouped) {
          if (int rc = select_group(l0, n)) return rc;
        } else {
          for (int l = l0; l < l0 + n; ++l)
            if (int rc = select(l)) return rc;
        }
      }
    }
    return NOSA_OK;
  };
  if (hio) {
    CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->in_stream, ctx->ev_fork, 0));
    CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->d2h_stream, ctx->ev_fork, 0));
  }
  // with the copy-engine mover, only the first two groups' inputs go ahead of the first miss
  // transfer; the rest follow it (the host submits that transfer once layer 0 is planned)
  if (int rc = issue_groups(groups.size())) return rc;
  // attention batches: att_plan's consecutive layer ranges, one persistent launch each
  // (layer-serial: one layer per launch, since select(l+1) waits for layer l to finish)
  std::vector<int>& att_l0 = ctx->att_l0;  // first layer of the batch that layer l closes, or -1
  att_l0.assign(dv.L, -1);
  if (serial) {
    for (int l = 0; l < dv.L; ++l) att_l0[l] = l;
  } else {
    for (int l0 = 0, k = 0; l0 < dv.L; l0 += ctx->att_plan[k++]) att_l0[l0 + ctx->att_plan[k] - 1] = l0;
  }
  int n_att = 0, n_gather_kernels = 0;
  ctx->memcpy_born_launches = 0;
  cudaEvent_t last_att[2] = {nullptr, nullptr};
  // hybrid mover: the SM share of every attention batch, device-driven on its own stream, queued
  // up front (each waits for its batch's last plan); the host packs the rest in the loop below
  auto smg_launch = [&](int l) -> int {
    const int l0 = ctx->att_l0[l];
    CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->smg_stream, ctx->ev_plan[l], 0));
    CUDA_TRY(ctx, nosa::launch_gather(dv, l0, ctx->smg_stream, ctx->gather_grid, false, l - l0 + 1));
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev_smg[l], ctx->smg_stream));
    ++n_gather_kernels;
    return NOSA_OK;
  };
  if (hybrid && !serial)
    for (int l = 0; l < dv.L; ++l)
      if (ctx->att_l0[l] >= 0)
        if (int rc = smg_launch(l)) return rc;
  for (int l = 0; l < dv.L; ++l) {
    if (serial) {
      if (l > 0) CUDA_TRY(ctx, cudaStreamWaitEvent(ss, ctx->ev_fin[l - 1], 0));
      if (int rc = project(l, 1)) return rc;
      if (int rc = select(l)) return rc;
    }
    const bool batch_end = att_l0[l] >= 0;  // last layer of an attention batch
    const int l0 = batch_end ? att_l0[l] : l, n = l - l0 + 1;
    if (!dv.born_local) {  // (all resident: the planner placed the newborn blocks, nothing to move)
      CUDA_TRY(ctx, cudaStreamWaitEvent(cp, ctx->ev_plan[l], 0));
      if (hostpack) {  // (records ev_gather[l] on the scatter stream itself)
        if (hybrid && batch_end) {
          if (serial)
            if (int rc = smg_launch(l)) return rc;
          CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->scatter_stream, ctx->ev_smg[l], 0));
        }
        if (int rc = gather_hostpack(ctx, l, cp, timed, hybrid)) return rc;
      } else if (io->gather_mode == NOSA_GATHER_MEMCPY) {
        const int rc = export_misses ? gather_exported(ctx, l, cp, timed) : gather_memcpy(ctx, l, ctx->ev_plan[l], cp, timed);
        if (rc) return rc;
      } else if (batch_end) {  // device movers: one launch for the attention batch's layers
        TimeScope ts(ctx, cp, 1, timed);
        const bool tma = io->gather_mode == NOSA_GATHER_TMA;
        CUDA_TRY(ctx, nosa::launch_gather(dv, l0, cp, tma ? ctx->tma_gather_grid : ctx->gather_grid, tma, n));
        ++n_gather_kernels;
      }
      if (!hostpack) CUDA_TRY(ctx, cudaEventRecord(ctx->ev_gather[l], cp));
    }
    if (!batch_end) continue;
    cudaStream_t a = (n_att & 1) ? at2 : at;
    // gathers run in order on cp; without gathers the plans complete in layer order on ss
    CUDA_TRY(ctx, cudaStreamWaitEvent(a, dv.born_local ? ctx->ev_plan[l] : ctx->ev_gather[l], 0));
    // record buffers: layer l' uses buffer l' % nbuf, last written for layer l' - nbuf
    if (l - dv.nbuf >= 0) CUDA_TRY(ctx, cudaStreamWaitEvent(a, ctx->ev_fin[l - dv.nbuf], 0));
    // Instrumented steps only: the batch's start event also waits for the previous batch (on the
    // other attention stream), whose persistent CTAs hold every SM until they retire, so the
    // event pair brackets this launch rather than its queueing behind the previous one.
    if (n_att > 0 && (timed || (ctx->capturing && ctx->cap_used < ctx->cap_events.size())))
      CUDA_TRY(ctx, cudaStreamWaitEvent(a, last_att[(n_att - 1) & 1], 0));
    {
      TimeScope ts(ctx, a, 2, timed);
      CUDA_TRY(ctx, nosa::launch_attend(dv, l0, n, q + l0 * qstride, kn + l0 * kstride, vn + l0 * kstride,
                                        io->out + l0 * ostride, a, ctx->num_sms));
    }
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev_att[l], a));
    last_att[n_att & 1] = ctx->ev_att[l];
    ++n_att;
    CUDA_TRY(ctx, cudaStreamWaitEvent(fn, ctx->ev_att[l], 0));
    {  // merge + append of the batch's layers in one launch
      TimeScope ts(ctx, fn, 3, timed);
      CUDA_TRY(ctx, nosa::launch_finalize(dv, l0, kn + l0 * kstride, vn + l0 * kstride, io->out + l0 * ostride, fn, n));
    }
    for (int lf = l0; lf <= l; ++lf) CUDA_TRY(ctx, cudaEventRecord(ctx->ev_fin[lf], fn));
    if (hio) {
      CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->d2h_stream, ctx->ev_fin[l], 0));
      TimeScope ts(ctx, ctx->d2h_stream, 5, timed);
      CUDA_TRY(ctx, cudaMemcpyAsync(hio->out + l0 * ostride, io->out + l0 * ostride, n * ostride * sizeof(float),
                                    cudaMemcpyDeviceToHost, ctx->d2h_stream));
    }
  }
  if (hio) {
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev_d2h, ctx->d2h_stream));
    CUDA_TRY(ctx, cudaStreamWaitEvent(st, ctx->ev_d2h, 0));
  }
  // join every side stream back into the caller's stream (the plans precede the last gather)
  CUDA_TRY(ctx, cudaStreamWaitEvent(st, ctx->ev_plan[dv.L - 1], 0));
  if (dv.born_local) CUDA_TRY(ctx, cudaEventRecord(ctx->ev_gather[dv.L - 1], cp));  // (no gathers: joins cp)
  CUDA_TRY(ctx, cudaStreamWaitEvent(st, ctx->ev_gather[dv.L - 1], 0));
  for (cudaEvent_t e : last_att)
    if (e) CUDA_TRY(ctx, cudaStreamWaitEvent(st, e, 0));
  CUDA_TRY(ctx, cudaStreamWaitEvent(st, ctx->ev_fin[dv.L - 1], 0));
  // kernels of this step: selections (grouped, per layer, or per layer + shared planner),
  // gathers (device movers), attention batches, finalizes, input staging (counted inline)
  const int n_sel = grouped ? (int)groups.size() * sel_kernels(dv) : (sel_kernels(dv) + (dv.shared ? 1 : 0)) * dv.L;
  ctx->step_kernels = n_sel + n_gather_kernels + ctx->memcpy_born_launches + 2 * n_att + n_proj;  // one finalize per attention batch
  if (count) ctx->launches += ctx->step_kernels;
  return NOSA_OK;
}

extern "C" int nosa_decode_step(NosaCtx* ctx, const NosaStepIO* io, void* stream) {
  if (!ctx || !io || !io->q || !io->k_new || !io->v_new || !io->out)
    return fail(ctx, NOSA_ERR_VALUE, "decode_step: NULL io");
  if (io->selector != 0 && io->selector != 1) return fail(ctx, NOSA_ERR_VALUE, "selector must be nosa or infllmv2");
  cudaSetDevice(ctx->device);
  return enqueue_step(ctx, io, S(stream), true);
}

// device staging of the host-buffer step: allocated on first use, `io` pointed at it
static int host_staging(NosaCtx* ctx, const NosaHostStepIO* hio, NosaStepIO* io_out) {
  if (!hio || !hio->q || !hio->k_new || !hio->v_new || !hio->out)
    return fail(ctx, NOSA_ERR_VALUE, "decode_step_host: NULL io");
  if (hio->selector != 0 && hio->selector != 1) return fail(ctx, NOSA_ERR_VALUE, "selector must be nosa or infllmv2");
  cudaSetDevice(ctx->device);
  const Dev& dv = ctx->dv;
  const size_t qb = (size_t)dv.L * dv.B * dv.Hq * dv.D * dv.elem, kb = (size_t)dv.L * dv.B * dv.H * dv.D * dv.elem;
  const size_t ob = (size_t)dv.L * dv.B * dv.Hq * dv.D * sizeof(float);
  const size_t need = qb + 2 * kb + ob;
  if (!ctx->io_buf) {
    CUDA_TRY(ctx, cudaMalloc(reinterpret_cast<void**>(&ctx->io_buf), need));
    ctx->io_bytes = need;
    CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->d2h_stream, cudaStreamNonBlocking));
    int prio_low = 0, prio_high = 0;
    cudaDeviceGetStreamPriorityRange(&prio_low, &prio_high);
    CUDA_TRY(ctx, cudaStreamCreateWithPriority(&ctx->in_stream, cudaStreamNonBlocking, prio_high));
    CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->ev_d2h, cudaEventDisableTiming));
    ctx->ev_in.resize(dv.L);
    for (int l = 0; l < dv.L; ++l) CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->ev_in[l], cudaEventDisableTiming));
  }
  NosaStepIO& io = *io_out;
  io = NosaStepIO{};
  io.q = ctx->io_buf;
  io.k_new = ctx->io_buf + qb;
  io.v_new = ctx->io_buf + qb + kb;
  io.out = reinterpret_cast<float*>(ctx->io_buf + qb + 2 * kb);
  io.selector = hio->selector;
  io.gather_mode = hio->gather_mode;
  io.schedule = hio->schedule;
  return NOSA_OK;
}

extern "C" int nosa_decode_step_host(NosaCtx* ctx, const NosaHostStepIO* hio, void* stream) {
  if (!ctx) return NOSA_ERR_VALUE;
  NosaStepIO io;
  if (int rc = host_staging(ctx, hio, &io)) return rc;
  return enqueue_step(ctx, &io, S(stream), true, hio);
}

extern "C" int nosa_set_projection(NosaCtx* ctx, int layer, const void* w_t, int d, int n, int nq, int nk) {
  int rc = check_layer(ctx, layer);
  if (rc) return rc;
  const Dev& dv = ctx->dv;
  if (dv.dtype != NOSA_DTYPE_BF16) return fail(ctx, NOSA_ERR_VALUE, "set_projection: the hidden-state step needs bf16 storage");
  if (!w_t) return fail(ctx, NOSA_ERR_VALUE, "set_projection: NULL weights");
  if (n != (dv.Hq + 2 * dv.H) * dv.D || nq != dv.Hq * dv.D || nk != dv.H * dv.D)
    return fail(ctx, NOSA_ERR_VALUE, "set_projection: weights must be [n_head + 2 n_kv_head] x d_head columns");
  if (d <= 0 || d % 64 || n % 128) return fail(ctx, NOSA_ERR_VALUE, "set_projection: needs d %% 64 == 0 and n %% 128 == 0");
  if (ctx->proj_d && d != ctx->proj_d) return fail(ctx, NOSA_ERR_VALUE, "set_projection: every layer needs the same d");
  cudaSetDevice(ctx->device);
  const size_t slab = (size_t)n * d * 2;
  if (!ctx->proj_wbuf) {
    CUDA_TRY(ctx, cudaMalloc(reinterpret_cast<void**>(&ctx->proj_wbuf), slab * dv.L));
    ctx->proj_set.assign(dv.L, 0);
  }
  CUDA_TRY(ctx, cudaMemcpy(ctx->proj_wbuf + layer * slab, w_t, slab, cudaMemcpyDefault));
  ctx->proj_set[layer] = 1;
  ctx->proj_d = d;
  return NOSA_OK;
}

static int hidden_staging(NosaCtx* ctx, const NosaHiddenStepIO* hid, NosaStepIO* io) {
  if (!hid || !hid->h || !hid->out) return fail(ctx, NOSA_ERR_VALUE, "decode_step_hidden: NULL io");
  if (ctx->proj_set.size() != (size_t)ctx->dv.L ||
      std::any_of(ctx->proj_set.begin(), ctx->proj_set.end(), [](char set) { return !set; }))
    return fail(ctx, NOSA_ERR_STATE, "decode_step_hidden: nosa_set_projection missing for a layer");
  NosaHostStepIO tmp{};  // device staging of q/k/v (the host-step buffers), `out` is the caller's
  tmp.q = tmp.k_new = tmp.v_new = hid->h;
  tmp.out = hid->out;
  tmp.selector = hid->selector;
  tmp.gather_mode = hid->gather_mode;
  tmp.schedule = hid->schedule;
  if (int rc = host_staging(ctx, &tmp, io)) return rc;
  io->out = hid->out;
  return NOSA_OK;
}

extern "C" int nosa_decode_step_hidden(NosaCtx* ctx, const NosaHiddenStepIO* hid, void* stream) {
  if (!ctx) return NOSA_ERR_VALUE;
  NosaStepIO io;
  if (int rc = hidden_staging(ctx, hid, &io)) return rc;
  return enqueue_step(ctx, &io, S(stream), true, nullptr, hid->h);
}
extern "C" int nosa_decode_step_hidden_host(NosaCtx* ctx, const NosaHiddenStepIO* hid, void* stream) {
  if (!ctx) return NOSA_ERR_VALUE;
  NosaStepIO io;
  if (int rc = hidden_staging(ctx, hid, &io)) return rc;
  // device copies: q/k/v and outputs in the host-step staging, h in its own buffer
  const Dev& dv = ctx->dv;
  const size_t hb = (size_t)dv.L * dv.B * ctx->proj_d * 2;
  if (ctx->hid_bytes < hb) {
    if (ctx->hid_buf) cudaFree(ctx->hid_buf);
    ctx->hid_buf = nullptr;
    CUDA_TRY(ctx, cudaMalloc(reinterpret_cast<void**>(&ctx->hid_buf), hb));
    ctx->hid_bytes = hb;
  }
  io.out = reinterpret_cast<float*>(ctx->io_buf + ctx->io_bytes - (size_t)dv.L * dv.B * dv.Hq * dv.D * sizeof(float));
  NosaHostStepIO out_only{};  // outputs back per attention batch (the host-step D2H path)
  out_only.out = hid->out;
  out_only.selector = hid->selector;
  out_only.gather_mode = hid->gather_mode;
  out_only.schedule = hid->schedule;
  return enqueue_step(ctx, &io, S(stream), true, &out_only, ctx->hid_buf, hid->h);
}

// device-visible aliases of pinned host buffers (NULL when a buffer is pageable)
static bool mapped_alias(const void* p, const char** out) {
  cudaPointerAttributes pa{};
  if (cudaPointerGetAttributes(&pa, p) != cudaSuccess || pa.type != cudaMemoryTypeHost || !pa.devicePointer) {
    cudaGetLastError();
    return false;
  }
  *out = static_cast<const char*>(pa.devicePointer);
  return true;
}

// CUDA graph of the host-buffer step (device movers only).  The host buffers of a replay may
// differ from the captured ones: the input-staging kernel nodes and the output copy nodes are
// re-pointed in the executable graph before the launch (launches already in flight keep theirs).
extern "C" int nosa_step_graph_capture_host(NosaCtx* ctx, const NosaHostStepIO* hio) {
  if (!ctx) return NOSA_ERR_VALUE;
  if (hio && (hio->gather_mode == NOSA_GATHER_MEMCPY || hio->gather_mode >= NOSA_GATHER_HOSTPACK))
    return fail(ctx, NOSA_ERR_VALUE, "graph capture needs a device-driven gather (uva or tma)");
  NosaStepIO io;
  if (int rc = host_staging(ctx, hio, &io)) return rc;
  const char* hs[3];
  if (ctx->stage_with_copies || !mapped_alias(hio->q, &hs[0]) || !mapped_alias(hio->k_new, &hs[1]) ||
      !mapped_alias(hio->v_new, &hs[2]))
    return fail(ctx, NOSA_ERR_VALUE, "graph host step needs pinned (mapped) input buffers");
  if (ctx->graph_exec_host) { cudaGraphExecDestroy(ctx->graph_exec_host); ctx->graph_exec_host = nullptr; }
  if (ctx->graph_host) { cudaGraphDestroy(ctx->graph_host); ctx->graph_host = nullptr; }
  ctx->capturing = false;
  CUDA_TRY(ctx, cudaStreamBeginCapture(ctx->capture_stream, cudaStreamCaptureModeThreadLocal));
  int rc = enqueue_step(ctx, &io, ctx->capture_stream, false, hio);
  cudaError_t e = cudaStreamEndCapture(ctx->capture_stream, &ctx->graph_host);
  if (rc) return rc;
  if (e != cudaSuccess) return fail(ctx, NOSA_ERR_CUDA, "stream capture: %s", cudaGetErrorString(e));
  CUDA_TRY(ctx, cudaGraphInstantiate(&ctx->graph_exec_host, ctx->graph_host, 0));
  ctx->graph_host_kernels = ctx->step_kernels + (int)ctx->groups.size();  // + one staging kernel per group
  // the nodes that hold host addresses
  ctx->host_nodes.clear();
  size_t n = 0;
  CUDA_TRY(ctx, cudaGraphGetNodes(ctx->graph_host, nullptr, &n));
  std::vector<cudaGraphNode_t> nodes(n);
  CUDA_TRY(ctx, cudaGraphGetNodes(ctx->graph_host, nodes.data(), &n));
  for (cudaGraphNode_t nd : nodes) {
    cudaGraphNodeType ty;
    CUDA_TRY(ctx, cudaGraphNodeGetType(nd, &ty));
    if (ty == cudaGraphNodeTypeKernel) {
      cudaKernelNodeParams kp{};
      CUDA_TRY(ctx, cudaGraphKernelNodeGetParams(nd, &kp));
      if (kp.func == nosa::stage_inputs_kernel_fn()) ctx->host_nodes.push_back({nd, 0});
    } else if (ty == cudaGraphNodeTypeMemcpy) {
      ctx->host_nodes.push_back({nd, 1});
    }
  }
  ctx->cap_hs[0] = hs[0]; ctx->cap_hs[1] = hs[1]; ctx->cap_hs[2] = hs[2];
  ctx->cap_out = hio->out;
  ctx->cur_hs[0] = hs[0]; ctx->cur_hs[1] = hs[1]; ctx->cur_hs[2] = hs[2];
  ctx->cur_out = hio->out;
  return NOSA_OK;
}

extern "C" int nosa_step_graph_launch_host(NosaCtx* ctx, const NosaHostStepIO* hio, void* stream) {
  if (!ctx || !ctx->graph_exec_host) return fail(ctx, NOSA_ERR_STATE, "no captured host step graph");
  if (!hio || !hio->q || !hio->k_new || !hio->v_new || !hio->out) return fail(ctx, NOSA_ERR_VALUE, "NULL io");
  const char* hs[3];
  if (!mapped_alias(hio->q, &hs[0]) || !mapped_alias(hio->k_new, &hs[1]) || !mapped_alias(hio->v_new, &hs[2]))
    return fail(ctx, NOSA_ERR_VALUE, "graph host step needs pinned (mapped) input buffers");
  const bool moved = hs[0] != ctx->cur_hs[0] || hs[1] != ctx->cur_hs[1] || hs[2] != ctx->cur_hs[2] ||
                     hio->out != ctx->cur_out;
  if (moved) {  // re-point every host-address node at the new buffers (same offsets)
    for (const auto& hn : ctx->host_nodes) {
      if (hn.kind == 0) {
        cudaKernelNodeParams kp{};
        CUDA_TRY(ctx, cudaGraphKernelNodeGetParams(hn.node, &kp));  // the captured arguments
        nosa::StageSeg seg[3];
        for (int i = 0; i < 3; ++i) {
          seg[i] = *static_cast<const nosa::StageSeg*>(kp.kernelParams[i]);
          const char* src = reinterpret_cast<const char*>(seg[i].src);
          seg[i].src = reinterpret_cast<const int4*>(hs[i] + (src - ctx->cap_hs[i]));
        }
        void* args[3] = {&seg[0], &seg[1], &seg[2]};
        kp.kernelParams = args;
        kp.extra = nullptr;
        CUDA_TRY(ctx, cudaGraphExecKernelNodeSetParams(ctx->graph_exec_host, hn.node, &kp));
      } else {
        cudaMemcpy3DParms mp{};
        CUDA_TRY(ctx, cudaGraphMemcpyNodeGetParams(hn.node, &mp));
        char* dst = static_cast<char*>(mp.dstPtr.ptr);
        const size_t bytes = mp.extent.width * mp.extent.height * mp.extent.depth;
        char* ndst = reinterpret_cast<char*>(hio->out) + (dst - reinterpret_cast<char*>(ctx->cap_out));
        CUDA_TRY(ctx, cudaGraphExecMemcpyNodeSetParams1D(ctx->graph_exec_host, hn.node, ndst, mp.srcPtr.ptr, bytes,
                                                         cudaMemcpyDeviceToHost));
      }
    }
    ctx->cur_hs[0] = hs[0]; ctx->cur_hs[1] = hs[1]; ctx->cur_hs[2] = hs[2];
    ctx->cur_out = hio->out;
  }
  CUDA_TRY(ctx, cudaGraphLaunch(ctx->graph_exec_host, S(stream)));
  ctx->launches += ctx->graph_host_kernels;
  return NOSA_OK;
}

static int capture_step(NosaCtx* ctx, const NosaStepIO* io, const void* hidden);

extern "C" int nosa_step_graph_capture(NosaCtx* ctx, const NosaStepIO* io) {
  if (!ctx || !io) return NOSA_ERR_VALUE;
  return capture_step(ctx, io, nullptr);
}

extern "C" int nosa_step_graph_capture_hidden(NosaCtx* ctx, const NosaHiddenStepIO* hid) {
  if (!ctx) return NOSA_ERR_VALUE;
  NosaStepIO io;
  if (int rc = hidden_staging(ctx, hid, &io)) return rc;
  return capture_step(ctx, &io, hid->h);
}

static int capture_step(NosaCtx* ctx, const NosaStepIO* io, const void* hidden) {
  if (io->gather_mode == NOSA_GATHER_MEMCPY || io->gather_mode >= NOSA_GATHER_HOSTPACK)
    return fail(ctx, NOSA_ERR_VALUE, "graph capture needs a device-driven gather (uva or tma)");
  cudaSetDevice(ctx->device);
  for (cudaGraphExec_t* x : {&ctx->graph_exec, &ctx->graph_exec_timed})
    if (*x) { cudaGraphExecDestroy(*x); *x = nullptr; }
  for (cudaGraph_t* x : {&ctx->graph, &ctx->graph_timed})
    if (*x) { cudaGraphDestroy(*x); *x = nullptr; }
  auto capture = [&](bool instrumented, cudaGraph_t* g) -> int {
    ctx->cap_used = 0;
    ctx->capturing = instrumented;
    CUDA_TRY(ctx, cudaStreamBeginCapture(ctx->capture_stream, cudaStreamCaptureModeThreadLocal));
    int rc = enqueue_step(ctx, io, ctx->capture_stream, false, nullptr, hidden);
    cudaError_t e = cudaStreamEndCapture(ctx->capture_stream, g);
    ctx->capturing = false;
    if (rc) return rc;
    if (e != cudaSuccess) return fail(ctx, NOSA_ERR_CUDA, "stream capture: %s", cudaGetErrorString(e));
    return NOSA_OK;
  };
  // the clean graph: what a replay runs unless per-kernel timing is on
  if (int rc = capture(false, &ctx->graph)) return rc;
  CUDA_TRY(ctx, cudaGraphInstantiate(&ctx->graph_exec, ctx->graph, 0));
  ctx->graph_kernels = ctx->step_kernels;
  // the instrumented twin: an external event-record node around every kernel (placeholders)
  const size_t nslots = 5 * (size_t)ctx->dv.L;
  while (ctx->cap_events.size() < nslots) {
    NosaCtx::Timed t{};
    CUDA_TRY(ctx, cudaEventCreate(&t.a));
    CUDA_TRY(ctx, cudaEventCreate(&t.b));
    ctx->cap_events.push_back(t);
  }
  if (int rc = capture(true, &ctx->graph_timed)) return rc;
  cudaGraph_t g = ctx->graph_timed;
  CUDA_TRY(ctx, cudaGraphInstantiate(&ctx->graph_exec_timed, g, 0));
  // map every event-record node back to its timing scope
  ctx->ev_nodes.clear();
  ctx->nodes_on_pool = false;  // freshly instantiated: the nodes hold the placeholders
  size_t n = 0;
  CUDA_TRY(ctx, cudaGraphGetNodes(g, nullptr, &n));
  std::vector<cudaGraphNode_t> nodes(n);
  CUDA_TRY(ctx, cudaGraphGetNodes(g, nodes.data(), &n));
  for (cudaGraphNode_t nd : nodes) {
    cudaGraphNodeType ty;
    CUDA_TRY(ctx, cudaGraphNodeGetType(nd, &ty));
    if (ty != cudaGraphNodeTypeEventRecord) continue;
    cudaEvent_t ev;
    CUDA_TRY(ctx, cudaGraphEventRecordNodeGetEvent(nd, &ev));
    for (size_t i = 0; i < ctx->cap_used; ++i) {
      if (ctx->cap_events[i].a == ev) ctx->ev_nodes.push_back({nd, (int)i, 0});
      if (ctx->cap_events[i].b == ev) ctx->ev_nodes.push_back({nd, (int)i, 1});
    }
  }
  return NOSA_OK;
}

extern "C" int nosa_step_graph_launch(NosaCtx* ctx, void* stream) {
  if (!ctx || !ctx->graph_exec) return fail(ctx, NOSA_ERR_STATE, "no captured step graph");
  const size_t slots = ctx->cap_used;
  if (ctx->graph_exec_timed && slots && ctx->timing_used + slots <= ctx->timing.size()) {
    // time this replay per kernel: point the instrumented twin's nodes at fresh pool events
    for (const auto& en : ctx->ev_nodes) {
      NosaCtx::Timed& t = ctx->timing[ctx->timing_used + en.slot];
      t.kind = ctx->cap_events[en.slot].kind;
      CUDA_TRY(ctx, cudaGraphExecEventRecordNodeSetEvent(ctx->graph_exec_timed, en.node, en.end ? t.b : t.a));
    }
    ctx->timing_used += slots;
    ctx->nodes_on_pool = true;
    CUDA_TRY(ctx, cudaGraphLaunch(ctx->graph_exec_timed, S(stream)));
    ctx->launches += ctx->graph_kernels;
    return NOSA_OK;
  }
  CUDA_TRY(ctx, cudaGraphLaunch(ctx->graph_exec, S(stream)));
  ctx->launches += ctx->graph_kernels;
  return NOSA_OK;
}

extern "C" int nosa_select_scores(int n_prob, const double* s_q, const double* s_e, int stride,
                                  const int32_t* pool_lo, const int32_t* pool_hi, int m_q, int m_e, int selector,
                                  int32_t* out_q, int32_t* n_q, int32_t* out_e, int32_t* n_e, void* stream) {
  if (n_prob <= 0) return NOSA_OK;
  if (!s_q || !pool_lo || !pool_hi || !out_q || !n_q || !out_e || !n_e || (selector == 0 && !s_e))
    return fail(nullptr, NOSA_ERR_VALUE, "select_scores: NULL argument");
  if (m_q < 0 || m_e < 0 || stride <= 0) return fail(nullptr, NOSA_ERR_VALUE, "select_scores: bad budgets");
  cudaError_t e = nosa::launch_select_scores(n_prob, s_q, s_e, stride, pool_lo, pool_hi, m_q, m_e, selector, out_q,
                                             n_q, out_e, n_e, S(stream));
  if (e != cudaSuccess) return fail(nullptr, NOSA_ERR_CUDA, "select_scores: %s", cudaGetErrorString(e));
  return NOSA_OK;
}

// ---------------------------------------------------------------- readback
#define SYNC_OR_FAIL(ctx)                                                      \
  do {                                                                         \
    cudaSetDevice((ctx)->device);                                              \
    cudaError_t _e = cudaDeviceSynchronize();                                  \
    if (_e != cudaSuccess)                                                     \
      return fail(ctx, NOSA_ERR_CUDA, "device error: %s", cudaGetErrorString(_e)); \
  } while (0)

extern "C" int nosa_read_selection(NosaCtx* ctx, int layer, int cap, int32_t* bq, int32_t* nq, int32_t* be,
                                   int32_t* ne, int32_t* req, int32_t* nreq, double* s_q) {
  int rc = check_layer(ctx, layer);
  if (rc) return rc;
  SYNC_OR_FAIL(ctx);
  const Dev& dv = ctx->dv;
  const size_t BH = (size_t)dv.B * dv.H, off = (size_t)layer * BH;
  std::vector<int> tq(BH * dv.MQ), te(BH * dv.ME), tr(BH * dv.C), cq(BH), ce(BH), cr(BH);
  CUDA_TRY(ctx, cudaMemcpy(tq.data(), dv.sel_q + off * dv.MQ, tq.size() * 4, cudaMemcpyDeviceToHost));
  CUDA_TRY(ctx, cudaMemcpy(te.data(), dv.sel_e + off * dv.ME, te.size() * 4, cudaMemcpyDeviceToHost));
  CUDA_TRY(ctx, cudaMemcpy(tr.data(), dv.req + off * dv.C, tr.size() * 4, cudaMemcpyDeviceToHost));
  CUDA_TRY(ctx, cudaMemcpy(cq.data(), dv.n_selq + off, BH * 4, cudaMemcpyDeviceToHost));
  CUDA_TRY(ctx, cudaMemcpy(ce.data(), dv.n_sele + off, BH * 4, cudaMemcpyDeviceToHost));
  CUDA_TRY(ctx, cudaMemcpy(cr.data(), dv.n_req + off, BH * 4, cudaMemcpyDeviceToHost));
  for (size_t x = 0; x < BH; ++x) {
    if (nq) nq[x] = cq[x];
    if (ne) ne[x] = ce[x];
    if (nreq) nreq[x] = cr[x];
    for (int i = 0; i < cap; ++i) {
      if (bq) bq[x * cap + i] = i < cq[x] && i < dv.MQ ? tq[x * dv.MQ + i] : -1;
      if (be) be[x * cap + i] = i < ce[x] && i < dv.ME ? te[x * dv.ME + i] : -1;
      if (req) req[x * cap + i] = i < cr[x] && i < dv.C ? tr[x * dv.C + i] : -1;
    }
  }
  if (s_q) {
    if (dv.screen) {  // the hot path scored only the candidates: recompute every pool row in f64
      CUDA_TRY(ctx, nosa::launch_score_readback(dv, layer, nullptr));
      SYNC_OR_FAIL(ctx);
    }
    CUDA_TRY(ctx, cudaMemcpy(s_q, dv.s_q + off * dv.NB, BH * dv.NB * 8, cudaMemcpyDeviceToHost));
  }
  return NOSA_OK;
}

extern "C" int nosa_read_plan(NosaCtx* ctx, int layer, int32_t* fetch, int32_t* nf, int32_t* evict, int32_t* ne,
                              int32_t* nh) {
  int rc = check_layer(ctx, layer);
  if (rc) return rc;
  SYNC_OR_FAIL(ctx);
  const Dev& dv = ctx->dv;
  const size_t BH = (size_t)dv.B * dv.H, off = (size_t)layer * BH;
  std::vector<int> n(BH * 3);
  CUDA_TRY(ctx, cudaMemcpy(n.data(), dv.plan_n + off * 3, n.size() * 4, cudaMemcpyDeviceToHost));
  if (fetch) CUDA_TRY(ctx, cudaMemcpy(fetch, dv.plan_fetch + off * dv.C, BH * dv.C * 4, cudaMemcpyDeviceToHost));
  if (evict) CUDA_TRY(ctx, cudaMemcpy(evict, dv.plan_evict + off * dv.C, BH * dv.C * 4, cudaMemcpyDeviceToHost));
  for (size_t x = 0; x < BH; ++x) {
    if (nf) nf[x] = n[x * 3 + 0];
    if (ne) ne[x] = n[x * 3 + 1];
    if (nh) nh[x] = n[x * 3 + 2];
  }
  return NOSA_OK;
}

extern "C" int nosa_read_residency(NosaCtx* ctx, int layer, int seq, int head, int32_t* slot_of, int32_t* block_of) {
  int rc = check_layer(ctx, layer);
  if (rc) return rc;
  const Dev& dv = ctx->dv;
  if (seq < 0 || seq >= dv.B || head < 0 || head >= dv.H) return fail(ctx, NOSA_ERR_VALUE, "seq/head out of range");
  SYNC_OR_FAIL(ctx);
  const size_t lbh = ((size_t)layer * dv.B + seq) * dv.H + head;
  if (slot_of) CUDA_TRY(ctx, cudaMemcpy(slot_of, dv.slot_of + lbh * dv.NB, dv.NB * 4, cudaMemcpyDeviceToHost));
  if (block_of) CUDA_TRY(ctx, cudaMemcpy(block_of, dv.blk_of + lbh * dv.C, dv.C * 4, cudaMemcpyDeviceToHost));
  return NOSA_OK;
}

extern "C" int nosa_read_block_scores(NosaCtx* ctx, int layer, double* s_e_c) {
  int rc = check_layer(ctx, layer);
  if (rc) return rc;
  SYNC_OR_FAIL(ctx);
  const Dev& dv = ctx->dv;
  const size_t BH = (size_t)dv.B * dv.H;
  CUDA_TRY(ctx, cudaMemcpy(s_e_c, dv.se + (size_t)layer * BH * dv.NB, BH * dv.NB * 8, cudaMemcpyDeviceToHost));
  return NOSA_OK;
}

static int read_blocks(NosaCtx* ctx, const char* src_dev, int nblocks, std::vector<char>& out) {
  const Dev& dv = ctx->dv;
  char* tmp = nullptr;
  const size_t bytes = (size_t)nblocks * dv.bpb;
  CUDA_TRY(ctx, cudaMalloc(&tmp, std::max<size_t>(bytes, 16)));
  nosa::launch_unswizzle(src_dev, tmp, nblocks, dv.n_b, dv.D, dv.elem, 0);
  out.resize(bytes);
  cudaError_t e = cudaMemcpy(out.data(), tmp, bytes, cudaMemcpyDeviceToHost);
  cudaFree(tmp);
  if (e != cudaSuccess) return fail(ctx, NOSA_ERR_CUDA, "read_blocks: %s", cudaGetErrorString(e));
  return NOSA_OK;
}

extern "C" int nosa_read_kv(NosaCtx* ctx, int layer, int seq, int head, int t, void* k, void* v) {
  int rc = check_layer(ctx, layer);
  if (rc) return rc;
  const Dev& dv = ctx->dv;
  if (seq < 0 || seq >= dv.B || head < 0 || head >= dv.H) return fail(ctx, NOSA_ERR_VALUE, "seq/head out of range");
  if (t < 0 || t > dv.NB * dv.n_b) return fail(ctx, NOSA_ERR_VALUE, "t out of range");
  if (t == 0) return NOSA_OK;
  SYNC_OR_FAIL(ctx);
  const size_t lbh = ((size_t)layer * dv.B + seq) * dv.H + head;
  const int nblk = (t + dv.n_b - 1) / dv.n_b;
  std::vector<char> buf;
  rc = read_blocks(ctx, dv.host + lbh * dv.NB * dv.bpb, nblk, buf);
  if (rc) return rc;
  const size_t row = (size_t)dv.D * dv.elem;
  memcpy(k, buf.data(), (size_t)t * row);
  memcpy(v, buf.data() + (size_t)nblk * dv.n_b * row, (size_t)t * row);
  return NOSA_OK;
}

extern "C" int nosa_read_slot(NosaCtx* ctx, int layer, int seq, int head, int slot, void* kv) {
  int rc = check_layer(ctx, layer);
  if (rc) return rc;
  const Dev& dv = ctx->dv;
  if (seq < 0 || seq >= dv.B || head < 0 || head >= dv.H || slot < 0 || slot >= dv.C)
    return fail(ctx, NOSA_ERR_VALUE, "seq/head/slot out of range");
  SYNC_OR_FAIL(ctx);
  const size_t lbh = ((size_t)layer * dv.B + seq) * dv.H + head;
  std::vector<char> buf;
  rc = read_blocks(ctx, dv.pool + (lbh * dv.C + slot) * dv.bpb, 1, buf);
  if (rc) return rc;
  memcpy(kv, buf.data(), buf.size());
  return NOSA_OK;
}

extern "C" int nosa_read_stats(NosaCtx* ctx, int l0, int l1, int s0, int s1, NosaStats* out) {
  if (!ctx || !out) return NOSA_ERR_VALUE;
  const Dev& dv = ctx->dv;
  if (l0 < 0 || l1 > dv.L || l0 > l1 || s0 < 0 || s1 > dv.B || s0 > s1) return fail(ctx, NOSA_ERR_VALUE, "stats range");
  SYNC_OR_FAIL(ctx);
  const size_t LBH = (size_t)dv.L * dv.B * dv.H;
  std::vector<long long> st(LBH * nosa::ST_N);
  CUDA_TRY(ctx, cudaMemcpy(st.data(), dv.stats, st.size() * 8, cudaMemcpyDeviceToHost));
  memset(out, 0, sizeof(*out));
  for (int l = l0; l < l1; ++l)
    for (int s = s0; s < s1; ++s)
      for (int h = 0; h < dv.H; ++h) {
        const long long* p = &st[(((size_t)l * dv.B + s) * dv.H + h) * nosa::ST_N];
        out->hits += p[nosa::ST_HITS];
        out->misses += p[nosa::ST_MISSES];
        out->new_blocks += p[nosa::ST_NEW];
        out->evictions += p[nosa::ST_EVICT];
        out->steps += p[nosa::ST_STEPS];
        out->candidates += p[nosa::ST_CAND];
        out->topk_required += p[nosa::ST_TOPK];
        out->topk_misses += p[nosa::ST_TOPK_MISS];
      }
  out->bytes_up = out->misses * dv.bpb;
  out->bytes_down = out->evictions * dv.bpb;
  return NOSA_OK;
}

extern "C" int nosa_reset_stats(NosaCtx* ctx, void* stream) {
  if (!ctx) return NOSA_ERR_VALUE;
  cudaSetDevice(ctx->device);
  CUDA_TRY(ctx, cudaMemsetAsync(ctx->dv.stats, 0, (size_t)ctx->dv.L * ctx->dv.B * ctx->dv.H * nosa::ST_N * 8, S(stream)));
  return NOSA_OK;
}

extern "C" int nosa_read_lengths(NosaCtx* ctx, int32_t* t) {
  if (!ctx || !t) return NOSA_ERR_VALUE;
  SYNC_OR_FAIL(ctx);
  const Dev& dv = ctx->dv;
  std::vector<int> all((size_t)dv.L * dv.B * dv.H);
  CUDA_TRY(ctx, cudaMemcpy(all.data(), dv.t, all.size() * 4, cudaMemcpyDeviceToHost));
  for (int l = 0; l < dv.L; ++l)
    for (int b = 0; b < dv.B; ++b) t[l * dv.B + b] = all[((size_t)l * dv.B + b) * dv.H];
  return NOSA_OK;
}

extern "C" int nosa_check_errors(NosaCtx* ctx, uint32_t* flags) {
  if (!ctx) return NOSA_ERR_VALUE;
  SYNC_OR_FAIL(ctx);
  unsigned f = 0;
  CUDA_TRY(ctx, cudaMemcpy(&f, ctx->dv.err, 4, cudaMemcpyDeviceToHost));
  if (flags) *flags = f;
  if (f) {
    cudaMemset(ctx->dv.err, 0, 4);
    if (f & NOSA_FLAG_CAPACITY)
      return fail(ctx, NOSA_ERR_CAPACITY, "step requires more blocks than the fast tier holds per head (%d)", ctx->dv.C);
    if (f & NOSA_FLAG_FULL)
      return fail(ctx, NOSA_ERR_VALUE, "head cache capacity exhausted (%d blocks of %d tokens); append refused",
                  ctx->dv.NB, ctx->dv.n_b);
    if (f & NOSA_FLAG_NOT_RESIDENT)
      return fail(ctx, NOSA_ERR_STATE, "all-resident run met a miss that is not a newborn block (flags 0x%x)", f);
    return fail(ctx, NOSA_ERR_VALUE, "device error flags 0x%x", f);
  }
  return NOSA_OK;
}
