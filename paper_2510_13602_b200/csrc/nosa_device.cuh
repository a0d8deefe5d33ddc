// nosa_device.cuh — device-side state layout and sm_100a helpers shared by the kernels.
//
// HBM / host layout (one "lbh" = (layer, sequence, kv head), lbh = (l * B + b) * H + h):
//   pool     [lbh][C][2][n_b][D]   HBM slot pool (fast tier).  One block = K plane then V plane,
//                                  bytes_per_block = 2*n_b*D*elem (kv_manager.py:78-81).
//   host     [lbh][NB][2][n_b][D]  pinned + mapped host mirror (slow tier, inclusive: it always
//                                  holds every block, so eviction is metadata only).
//   Within each K/V plane, the 16-byte chunk c of row r is stored at chunk c ^ (r & 7) so that
//   ldmatrix row gathers of 8 rows hit 8 distinct bank groups (storage format, not semantics).
//   kc       [lbh][NB][D]  f64     block-mean keys of complete blocks (compress_blocks)
//   se       [lbh][NB]     f64     block-mean importance score of complete blocks
//   tail_*                         running sums of the partial tail block
//   slot_of  [lbh][NB]  i32        block -> slot (-1 = slow only)      (TieredBlockManager.table)
//   blk_of / lastreq / fstack [lbh][C]  slot -> block, last-required clock, LIFO free stack
#pragma once
#include <cuda_runtime.h>
#include <cstdlib>
#include <cuda_bf16.h>
#include <stdint.h>

namespace nosa {

constexpr int kChunk = 8;  // max KV blocks per attention work item (split-K granularity)
constexpr int kCntStride = 4;  // ints per layer in Dev::cnt

struct Dev {
  // ---- shapes --------------------------------------------------------------------------
  int B, H, Hq, G, D, n_b, n_s, n_w, n_sink;
  int m_q, m_e, m_topk, MQ, ME;  // blocks_q, blocks_e, blocks_topk; selection capacities
  int L, C, NB, n_ev;            // layers, fast slots, max blocks, eviction-head width (n_head)
  int dtype, variant, elem;
  int shared;                    // 1: one fast pool of B*C slots per (layer, head) shared by the batch
                                 //    (the reference simulator, offload_sim.py:254-256); slot_of then
                                 //    holds the shared slot id s, stored at (lbh of batch s/C, slot s%C)
  long long bpb;                 // bytes per block
  int chunk;                     // KV blocks per attention work item, 1..kChunk
  int max_chunks;                // ceil(C / chunk)
  int nbuf;                      // split-K record buffers (layer l uses buffer l % nbuf)
  // ---- persistent state ----------------------------------------------------------------
  char* pool;
  char* host;                    // device-visible alias of the pinned host mirror
  double* kc;
  double* se;
  double* tail_ksum;
  double* tail_se;
  int* rank_e;
  int* slot_of;
  int* blk_of;
  int* lastreq;
  int* fstack;
  int* ftop;
  int* clock;
  int* t;
  int* t0;
  long long* stats;              // [lbh][8]: hits, misses, new, evictions, steps
  // ---- per-step buffers ----------------------------------------------------------------
  int* req;                      // [lbh][C]
  int* req_slot;                 // [lbh][C]
  int* n_req;                    // [lbh]
  int* sel_q;                    // [lbh][MQ]
  int* n_selq;
  int* sel_e;                    // [lbh][ME]
  int* n_sele;
  double* s_q;                   // [lbh][NB] pool scores (kept for parity readback)
  // ---- screened selection (exact top-k from a bf16 pre-scan + f64 refinement) -----------
  int screen;                    // 1: screened scan (default), 0: full f64 scan of the pool
  int born_local;                // 1: every block is HBM-resident for the run, so a block born by an
                                 // append is the only miss; the planner rebuilds it and no gather runs
  __nv_bfloat16* kc16;           // [lbh][NB][D] bf16(K_c) of the frozen pool (built at start_run)
  float* kc_err;                 // [lbh][NB] sum_i |K_c - bf16(K_c)| of each pool row (rounded up)
  double* qsum_buf;              // [lbh][D] the step's q_sum (parity readback recomputes s_q)
  int split_scan;                // 1: the screen scan is its own bandwidth-bound kernel ahead of
                                 // the selection/planning kernel (default), 0: fused in select_plan
  unsigned* scr_lo;              // [lbh][NB] screened lower bound of each pool row (monotone key)
  float* scr_up;                 // [lbh][NB] screened upper bound
  int* plan_fetch;               // [lbh][C]
  int* plan_evict;               // [lbh][C]
  int* plan_n;                   // [lbh][3] n_fetch, n_evict, n_hit
  int* cnt;                      // [L][kCntStride]: miss count, attention work counter, exported
                                 // (copy-engine) misses, plan CTAs done
  // copy-engine miss export (NOSA_GATHER_MEMCPY inside a step): the planner writes each layer's
  // copy list straight into mapped pinned host memory, so the host submits the batch with no
  // device round trip (nosa_ctx.cu gather_exported)
  int x_on;                      // set per launch: export this launch's misses
  int x_split;                   // host-pack share (hybrid mover): units with unit_hash < x_split
                                 // go to the exported list, the rest stay with the SM gather; 1024 = all
  void** x_src;                  // [L][B*H*C] device alias of the host array of source addresses
  void** x_dst;                  // [L][B*H*C] destination slot addresses
  int* x_cnt;                    // [L][2] device alias of host ints: exported misses, born blocks
  const char* x_src_base;        // slow-tier base address as the copy engine sees it
  int4* miss_list;               // [L][B*H*C]  {lbh, blk, slot, 0}
  float* part_o;                 // [nbuf][B*H][max_chunks][G][D]  split-K records (layer % nbuf)
  float2* part_ml;               // [nbuf][B*H][max_chunks][G]     (m, l) of each record
  char* newrow;                  // [lbh][2][D] (elem): K and V row of the last block born by an append
  unsigned long long* ktime;     // diagnostics (NULL = off): [L][2] device-clock start/end of attention launches
  long long* sel_prof;           // diagnostics (NULL = off): [16] select_plan cycles per phase, [15] = CTAs
  double* w1;                    // [D][n_ev]
  double* w2;                    // [n_ev]
  unsigned* err;
};

// one host segment of the input-staging kernel (nosa_gather.cu); the host-step graph re-points
// `src` between replays (nosa_ctx.cu)
struct StageSeg {
  const int4* src;
  int4* dst;
  long long n16;
};

// ST_CAND: rows rescored in f64; ST_TOPK / ST_TOPK_MISS: required pool (top-k) blocks and the
// fetches among them (offload_sim.py:291-293, hit_rate_topk)
enum StatIdx { ST_HITS = 0, ST_MISSES, ST_NEW, ST_EVICT, ST_STEPS, ST_CAND, ST_TOPK, ST_TOPK_MISS, ST_N = 8 };

// shared-pool mode: storage index of shared slot s of (layer, head) in the [lbh][C] arrays, and
// the slot offset relative to sequence b's own pool row (pool + (lbh*C + rel)*bpb addresses it)
__host__ __device__ __forceinline__ size_t shared_idx(const Dev& dv, int layer, int h, int s) {
  return ((size_t)(layer * dv.B + s / dv.C) * dv.H + h) * dv.C + s % dv.C;
}
__host__ __device__ __forceinline__ int shared_rel(const Dev& dv, int b, int s) {
  return (s / dv.C - b) * dv.H * dv.C + s % dv.C;
}

// the split-K record buffer of a layer (nbuf buffers: attention batches are double-buffered)
__host__ __device__ __forceinline__ float* part_o_of(const Dev& dv, int layer) {
  return dv.part_o + (size_t)(layer % dv.nbuf) * dv.B * dv.H * dv.max_chunks * dv.G * dv.D;
}
__host__ __device__ __forceinline__ float2* part_ml_of(const Dev& dv, int layer) {
  return dv.part_ml + (size_t)(layer % dv.nbuf) * dv.B * dv.H * dv.max_chunks * dv.G;
}

// Every kernel of the step asks for the maximum shared-memory carveout, so an SM never has to
// change its L1/shared split (and drain its resident CTAs) between the persistent attention
// kernel and the kernels that run beside it.  NOSA_NO_CARVEOUT=1 turns this off (A/B).
template <typename F>
inline void max_shared_carveout(F* kernel) {
  static const bool on = getenv("NOSA_NO_CARVEOUT") == nullptr;
  if (on) cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}

// ---------------------------------------------------------------- small helpers
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// Total order on doubles matching numpy's comparisons for finite / inf values, with -0.0
// folded onto +0.0 (argtopk treats them as equal, numerics.py:72).  Larger key = larger score.
__device__ __forceinline__ unsigned long long order_key(double s) {
  if (s == 0.0) s = 0.0;
  unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(s));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// byte offset of element (row r, col c) inside one [n_b][D] plane in the swizzled format
__device__ __forceinline__ int swz_off(int r, int c, int D, int elem) {
  const int row_bytes = D * elem;
  const int byte = c * elem;
  const int chunk = (byte >> 4) ^ (r & 7);
  return r * row_bytes + (chunk << 4) + (byte & 15);
}

// ---------------------------------------------------------------- mbarrier / bulk copy PTX
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// 1-D bulk copy global -> shared, completion counted on `bar` (TMA engine, SASS UBLKCP)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_plain(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// ---------------------------------------------------------------- warp-level tensor-core PTX
__device__ __forceinline__ void ldsm_x4(unsigned addr, unsigned& r0, unsigned& r1, unsigned& r2,
                                        unsigned& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(unsigned addr, unsigned& r0, unsigned& r1,
                                          unsigned& r2, unsigned& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
// D = A(16x16 bf16, row) * B(16x8 bf16, col) + C, fp32 accumulate
__device__ __forceinline__ void mma_bf16(float (&c)[4], unsigned a0, unsigned a1, unsigned a2,
                                         unsigned a3, unsigned b0, unsigned b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ unsigned pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<unsigned*>(&v);
}

template <typename T>
__device__ __forceinline__ double to_f64(T x);
template <>
__device__ __forceinline__ double to_f64<float>(float x) { return static_cast<double>(x); }
template <>
__device__ __forceinline__ double to_f64<__nv_bfloat16>(__nv_bfloat16 x) {
  return static_cast<double>(__bfloat162float(x));
}
template <typename T>
__device__ __forceinline__ float to_f32(T x);
template <>
__device__ __forceinline__ float to_f32<float>(float x) { return x; }
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 x) {
  return __bfloat162float(x);
}

// silu in f64 with the reference's split sigmoid (attention.py:29-40)
__device__ __forceinline__ double silu64(double x) {
  double s;
  if (x >= 0.0) {
    s = 1.0 / (1.0 + exp(-x));
  } else {
    const double e = exp(x);
    s = e / (1.0 + e);
  }
  return x * s;
}

// importance score of one token from its value row (importance_scores, attention.py:121-146):
// z = silu(v W1) W2 (ed-dma / s-dma), exp(z) (dma).  Executed by one warp; returns on all lanes.
template <typename T>
__device__ double token_score_warp(const T* v, const double* w1, const double* w2, int D,
                                   int n_ev, int variant) {
  const int lane = threadIdx.x & 31;
  double z = 0.0;
  for (int j = 0; j < n_ev; ++j) {
    double part = 0.0;
    for (int i = lane; i < D; i += 32) part = fma(to_f64(v[i]), w1[i * n_ev + j], part);
#pragma unroll
    for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    z = fma(silu64(part), w2[j], z);
  }
  return variant == 2 ? exp(z) : z;
}

// A block born by the previous step's append: row 0 from the device stash, zeros elsewhere
// (the miss gathers and, for all-resident runs, the planner)
__device__ __forceinline__ void write_born_block(const Dev& dv, int4 m, int4* dst, int vecs) {
  const int row_vecs = dv.D * dv.elem / 16, plane_vecs = vecs / 2;
  const int4* stash = reinterpret_cast<const int4*>(dv.newrow + (size_t)m.x * 2 * dv.D * dv.elem);
  for (int i = threadIdx.x; i < vecs; i += blockDim.x) {
    const int which = i / plane_vecs, in_plane = i - which * plane_vecs;
    dst[i] = in_plane < row_vecs ? stash[which * row_vecs + in_plane] : make_int4(0, 0, 0, 0);
  }
}

}  // namespace nosa
