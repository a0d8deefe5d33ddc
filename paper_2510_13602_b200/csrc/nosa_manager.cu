// nosa_manager.cu — the reference TieredBlockManager (kv_manager.py:130-363) with its tables in HBM.
//
// Exclusive two-tier residency exactly as the reference defines it: every logical key
// (batch, head, block) lives in one tier at a time, each tier keeps one LIFO free list per head
// (kv_manager.py:147-150), a plan fetches the required keys missing from FAST and evicts the
// least-recently-required non-required FAST keys of the head by (last_required, batch, block)
// (kv_manager.py:125-127, 205-259), and applying it moves evictions FAST -> SLOW, then fetches
// SLOW -> FAST, one _move at a time (kv_manager.py:261-298).
//
// Keys are addressed by a dense per-head id the host binding assigns at allocate() (its
// key -> id dict translates the reference's tuples); everything else -- tier / slot tables, the
// recency clock, the free lists, victim selection, the moves and the payload copies -- runs on
// the device, one CTA per call.  Victim selection is a radix select over the 96-bit key
// (last_required, batch, block) of every candidate in the head's FAST tier, so a 16K-slot shared
// pool plans in one pass instead of sorting every fast key (the reference's 5.5 ms per call).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/nosa_b200.h"

namespace {

constexpr int kThreads = 1024;
// status bits written by the kernels (host maps them to the reference exceptions)
constexpr int kErrCapacity = 1, kErrUnknown = 2, kErrEvictable = 4, kErrOutOfBlocks = 8, kErrDuplicate = 16;

struct Mgr {
  int H, F, S, ids;          // heads, fast slots / head, slow slots / head, id capacity / head (F + S)
  int8_t* tier;              // [H][ids]  -1 unmapped, 0 FAST, 1 SLOW
  int* slot;                 // [H][ids]
  unsigned* last;            // [H][ids]  last_required clock (0 = never; kv_manager.py:127 .get(key, 0))
  int2* kb;                  // [H][ids]  (batch, block) of the key
  int* fast_id;              // [H][F]    slot -> id (-1 free)
  int* slow_id;              // [H][S]
  int* fast_free;            // [H][F]    LIFO stacks, top = count
  int* slow_free;            // [H][S]
  int* tops;                 // [H][2]    fast, slow stack sizes
  unsigned* clock;           // [1]       the manager's plan clock (kv_manager.py:211)
  int* io;                   // call scratch (device): inputs and outputs of one call
  int* status;               // [1]
  // payload (store_payload): FAST in HBM, SLOW in mapped pinned host memory, reference layout
  // (num_blocks, heads, 2, n_b, d_head) per tier (kv_manager.py:161-166)
  char* pay_fast;
  char* pay_slow;            // device alias
  long long bpb;             // bytes per block
};

__device__ __forceinline__ void set_err(const Mgr& m, int bit) { atomicOr(m.status, bit); }

// allocate (kv_manager.py:171-183): tier 0/1, one key
__global__ void mgr_allocate_kernel(Mgr m, int h, int id, int tier, int batch, int block) {
  const size_t k = (size_t)h * m.ids + id;
  if (m.tier[k] >= 0) { set_err(m, kErrDuplicate); return; }
  int* top = m.tops + 2 * h + tier;
  if (*top == 0) { set_err(m, kErrOutOfBlocks); return; }
  const int s = (tier == 0 ? m.fast_free + (size_t)h * m.F : m.slow_free + (size_t)h * m.S)[--*top];
  m.tier[k] = (int8_t)tier;
  m.slot[k] = s;
  m.last[k] = 0u;
  m.kb[k] = make_int2(batch, block);
  (tier == 0 ? m.fast_id + (size_t)h * m.F : m.slow_id + (size_t)h * m.S)[s] = id;
  m.io[0] = s;
}

// free_block (kv_manager.py:185-194): the slot goes back on its tier's LIFO list, the key's
// recency is dropped
__global__ void mgr_free_kernel(Mgr m, int h, int id) {
  const size_t k = (size_t)h * m.ids + id;
  const int t = m.tier[k];
  if (t < 0) { set_err(m, kErrUnknown); return; }
  const int s = m.slot[k];
  if (t == 0) {
    m.fast_id[(size_t)h * m.F + s] = -1;
    m.fast_free[(size_t)h * m.F + m.tops[2 * h]++] = s;
  } else {
    m.slow_id[(size_t)h * m.S + s] = -1;
    m.slow_free[(size_t)h * m.S + m.tops[2 * h + 1]++] = s;
  }
  m.tier[k] = -1;
  m.last[k] = 0u;
}

// 96-bit victim key, most significant word first
struct VKey { unsigned w[3]; };
__device__ __forceinline__ VKey vkey(const Mgr& m, size_t k) {
  const int2 bb = m.kb[k];
  return {{m.last[k], (unsigned)bb.x ^ 0x80000000u, (unsigned)bb.y ^ 0x80000000u}};  // signed -> ordered
}
__device__ __forceinline__ bool vless(const VKey& a, const VKey& b) {
  for (int i = 0; i < 3; ++i)
    if (a.w[i] != b.w[i]) return a.w[i] < b.w[i];
  return false;
}

// plan_transfers (kv_manager.py:205-259) for one (batch, head) call.
// io in:  [0] n required, [1..n] ids in ascending block order (-1 = unmapped key)
// io out: base = 1 + n: [base] n_fetch, [base+1] n_evict, [base+2] hits,
//         fetch ids at base+3.., evict ids after them (victim order)
// policy != 0 (a caller-supplied eviction_policy, kv_manager.py:133-138): no victim choice; when
//         evictions are needed, the evictable candidates (kv_manager.py:236-243) follow the fetch
//         ids as [count][ids in fast-slot order] for the caller to order
__global__ void __launch_bounds__(kThreads) mgr_plan_kernel(Mgr m, int h, int batch, int policy) {
  __shared__ unsigned hist[256];
  __shared__ int s_cnt, s_nf, s_hits, s_digit, s_below, s_nv, s_unknown;
  __shared__ VKey s_thr;
  const int tid = threadIdx.x;
  const int n = m.io[0];
  const int* req = m.io + 1;
  int* out = m.io + 1 + n;
  const unsigned clock = m.clock[0] + 1;
  if (tid == 0) {
    m.clock[0] = clock;  // the tick happens before any check (kv_manager.py:211-212)
    s_cnt = 0;
    s_unknown = 0;
    s_nf = 0;
    s_hits = 0;
    out[0] = out[1] = out[2] = 0;
  }
  __syncthreads();
  if (n > m.F) {
    if (tid == 0) set_err(m, kErrCapacity);
    return;
  }
  // (1) required keys in block order: the first unmapped one raises UnknownKey after the
  //     recency of the keys before it was updated (the reference loop, kv_manager.py:219-229)
  if (tid == 0) {
    int nf = 0, hits = 0;
    for (int i = 0; i < n; ++i) {
      const int id = req[i];
      if (id < 0 || m.tier[(size_t)h * m.ids + id] < 0) {
        set_err(m, kErrUnknown);
        s_unknown = 1;  // (its own flag: s_cnt is reset below while others may still test this)
        break;
      }
      const size_t k = (size_t)h * m.ids + id;
      m.last[k] = clock;
      if (m.tier[k] == 0) ++hits;
      else out[3 + nf++] = id;
    }
    s_nf = nf;
    s_hits = hits;
  }
  __syncthreads();
  if (s_unknown) return;
  const int nf = s_nf;
  const int shortfall = nf - m.tops[2 * h];
  int* ev = out + 3 + nf;
  if (shortfall > 0 && policy) {
    if (tid == 0) {
      const int* fid = m.fast_id + (size_t)h * m.F;
      int nc = 0;
      for (int s = 0; s < m.F; ++s) {
        const int id = fid[s];
        if (id < 0) continue;
        const size_t k = (size_t)h * m.ids + id;
        if (!(m.last[k] == clock && m.kb[k].x == batch)) ev[1 + nc++] = id;
      }
      ev[0] = nc;
    }
  } else if (shortfall > 0) {
    // (2) candidates: FAST keys of the head not (batch == b and block in required): the
    //     required ids of this call carry last == clock and batch == b, so they are exactly the
    //     FAST keys with last == clock and kb.x == batch (a key of another batch keeps last <
    //     clock: one call per clock tick)
    const int* fid = m.fast_id + (size_t)h * m.F;
    auto is_cand = [&](int s, size_t& k) -> bool {
      const int id = fid[s];
      if (id < 0) return false;
      k = (size_t)h * m.ids + id;
      return !(m.last[k] == clock && m.kb[k].x == batch);
    };
    // radix select of the shortfall-th smallest key, 8 bits at a time over 96 bits
    VKey prefix = {{0u, 0u, 0u}};
    int want = shortfall;  // rank (1-based) of the threshold among candidates matching prefix
    if (tid == 0) s_cnt = 0;
    __syncthreads();
    for (int s = tid; s < m.F; s += kThreads) {
      size_t k;
      if (is_cand(s, k)) atomicAdd(&s_cnt, 1);
    }
    __syncthreads();
    if (s_cnt < shortfall) {  // kv_manager.py:246-250
      if (tid == 0) set_err(m, kErrEvictable);
      return;
    }
    for (int pass = 0; pass < 12; ++pass) {
      const int word = pass / 4, shift = 24 - 8 * (pass % 4);
      for (int i = tid; i < 256; i += kThreads) hist[i] = 0u;
      __syncthreads();
      for (int s = tid; s < m.F; s += kThreads) {
        size_t k;
        if (!is_cand(s, k)) continue;
        const VKey v = vkey(m, k);
        bool match = true;  // the digits above this one equal the prefix
        for (int p = 0; p < pass; ++p) {
          const int w = p / 4, sh = 24 - 8 * (p % 4);
          if (((v.w[w] >> sh) & 255u) != ((prefix.w[w] >> sh) & 255u)) { match = false; break; }
        }
        if (match) atomicAdd(&hist[(v.w[word] >> shift) & 255u], 1u);
      }
      __syncthreads();
      if (tid == 0) {
        int acc = 0, d = 0;
        for (; d < 256; ++d) {
          if (acc + (int)hist[d] >= want) break;
          acc += hist[d];
        }
        s_digit = d;
        s_below = acc;
      }
      __syncthreads();
      prefix.w[word] |= (unsigned)s_digit << shift;
      want -= s_below;
      __syncthreads();
    }
    // keys are unique per head, so the victims are exactly the candidates <= the threshold key
    if (tid == 0) {
      s_thr = prefix;
      s_nv = 0;
    }
    __syncthreads();
    // (3) victim order = rank among the victims (shortfall is small next to F)
    for (int s = tid; s < m.F; s += kThreads) {
      size_t k;
      if (!is_cand(s, k)) continue;
      const VKey v = vkey(m, k);
      if (vless(s_thr, v)) continue;
      int rank = 0;
      for (int u = 0; u < m.F; ++u) {
        size_t k2;
        if (u == s || !is_cand(u, k2)) continue;
        const VKey v2 = vkey(m, k2);
        if (!vless(s_thr, v2) && vless(v2, v)) ++rank;
      }
      ev[rank] = fid[s];
    }
    __syncthreads();
  }
  if (tid == 0) {
    out[0] = nf;
    out[1] = shortfall > 0 ? shortfall : 0;
    out[2] = s_hits;
  }
}

// apply_transfers' moves (kv_manager.py:276-298) in the reference order, one _move at a time
// (thread 0: each move pops the destination tier's LIFO list and pushes the source slot), then
// the payload copies, evictions before fetches (a fetch may land in a slot an eviction vacated).
// io in: [0] n_evict, [1] n_fetch, evict ids, fetch ids; out after them: src slot, dst slot per move
__global__ void __launch_bounds__(kThreads) mgr_apply_kernel(Mgr m, int h, int copy_payload) {
  const int ne = m.io[0], nf = m.io[1], nm = ne + nf;
  const int* ids = m.io + 2;
  int* mv = m.io + 2 + nm;  // [nm][2]
  if (threadIdx.x == 0) {
    for (int i = 0; i < nm; ++i) {
      const int id = ids[i];
      const size_t k = (size_t)h * m.ids + id;
      const int dst_tier = i < ne ? 1 : 0, src_tier = m.tier[k];
      const int src = m.slot[k];
      if (src_tier == dst_tier) {  // _move is a no-op (kv_manager.py:284-285)
        mv[2 * i] = mv[2 * i + 1] = -1;
        continue;
      }
      int* top = m.tops + 2 * h + dst_tier;
      if (*top == 0) {
        set_err(m, kErrOutOfBlocks);
        return;
      }
      const int dst = (dst_tier == 0 ? m.fast_free + (size_t)h * m.F : m.slow_free + (size_t)h * m.S)[--*top];
      m.tier[k] = (int8_t)dst_tier;
      m.slot[k] = dst;
      if (dst_tier == 0) {
        m.fast_id[(size_t)h * m.F + dst] = id;
        m.slow_id[(size_t)h * m.S + src] = -1;
        m.slow_free[(size_t)h * m.S + m.tops[2 * h + 1]++] = src;
      } else {
        m.slow_id[(size_t)h * m.S + dst] = id;
        m.fast_id[(size_t)h * m.F + src] = -1;
        m.fast_free[(size_t)h * m.F + m.tops[2 * h]++] = src;
      }
      mv[2 * i] = src;
      mv[2 * i + 1] = dst;
    }
  }
  if (!m.pay_fast || !copy_payload) return;
  __syncthreads();
  const int vecs = (int)(m.bpb / 16);
  for (int phase = 0; phase < 2; ++phase) {
    const int i0 = phase ? ne : 0, i1 = phase ? nm : ne;
    for (int i = i0; i < i1; ++i) {
      if (mv[2 * i] < 0) continue;
      const char* src = (phase ? m.pay_slow : m.pay_fast) + ((size_t)mv[2 * i] * m.H + h) * m.bpb;
      char* dst = (phase ? m.pay_fast : m.pay_slow) + ((size_t)mv[2 * i + 1] * m.H + h) * m.bpb;
      for (int v = threadIdx.x; v < vecs; v += kThreads)
        reinterpret_cast<int4*>(dst)[v] = reinterpret_cast<const int4*>(src)[v];
    }
    __syncthreads();
    __threadfence_system();
  }
}

// audit (kv_manager.py:341-363): per (tier, head) the mapped slots and the free list are disjoint
// and cover the tier's slots; the slot -> id maps agree with the key tables
__global__ void mgr_audit_kernel(Mgr m, int* bad) {
  const int h = blockIdx.x;
  for (int tier = 0; tier < 2; ++tier) {
    const int N = tier ? m.S : m.F;
    const int* sid = (tier ? m.slow_id + (size_t)h * m.S : m.fast_id + (size_t)h * m.F);
    const int* fr = (tier ? m.slow_free + (size_t)h * m.S : m.fast_free + (size_t)h * m.F);
    const int top = m.tops[2 * h + tier];
    for (int s = threadIdx.x; s < N; s += blockDim.x) {
      int in_free = 0;
      for (int i = 0; i < top; ++i) in_free += fr[i] == s;
      const int id = sid[s];
      if (id >= 0) {
        const size_t k = (size_t)h * m.ids + id;
        if (in_free || m.tier[k] != tier || m.slot[k] != s) atomicOr(bad, 1 << tier);
      } else if (in_free != 1) {
        atomicOr(bad, 4 << tier);
      }
    }
    for (int id = threadIdx.x; id < m.ids; id += blockDim.x) {
      const size_t k = (size_t)h * m.ids + id;
      if (m.tier[k] == tier && sid[m.slot[k]] != id) atomicOr(bad, 16 << tier);
    }
  }
}

}  // namespace

struct NosaMgr {
  Mgr m{};
  int device = 0;
  int n_b = 0, d_head = 0, elem = 0;
  std::vector<void*> allocs;
  char* host_pay = nullptr;
  int* h_io = nullptr;   // pinned mirror of m.io
  size_t io_ints = 0;
  cudaStream_t st = nullptr;
  std::string err;
};

static int mfail(NosaMgr* g, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (g) g->err = buf;
  return code;
}

#define MGR_TRY(g, expr)                                                                     \
  do {                                                                                       \
    cudaError_t _e = (expr);                                                                 \
    if (_e != cudaSuccess) {                                                                 \
      cudaGetLastError();                                                                    \
      return mfail(g, NOSA_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(_e));               \
    }                                                                                        \
  } while (0)

template <typename T>
static int malloc_zero(NosaMgr* g, T** p, size_t count, int fill_byte = 0) {
  MGR_TRY(g, cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(count, 1) * sizeof(T)));
  g->allocs.push_back(*p);
  MGR_TRY(g, cudaMemset(*p, fill_byte, std::max<size_t>(count, 1) * sizeof(T)));
  return NOSA_OK;
}

// runs the call's kernel and maps the status bits onto the reference exceptions
static int finish(NosaMgr* g, const char* what) {
  MGR_TRY(g, cudaGetLastError());
  int status = 0;
  MGR_TRY(g, cudaMemcpyAsync(&g->h_io[g->io_ints - 1], g->m.status, sizeof(int), cudaMemcpyDeviceToHost, g->st));
  MGR_TRY(g, cudaStreamSynchronize(g->st));
  status = g->h_io[g->io_ints - 1];
  if (!status) return NOSA_OK;
  MGR_TRY(g, cudaMemsetAsync(g->m.status, 0, sizeof(int), g->st));
  if (status & kErrCapacity) return mfail(g, NOSA_ERR_CAPACITY, "%s: the required set exceeds the fast tier", what);
  if (status & kErrEvictable) return mfail(g, NOSA_ERR_CAPACITY, "%s: not enough evictable fast blocks", what);
  if (status & kErrUnknown) return mfail(g, NOSA_ERR_UNKNOWN_KEY, "%s: key is not mapped", what);
  if (status & kErrOutOfBlocks) return mfail(g, NOSA_ERR_OUT_OF_BLOCKS, "%s: tier has no free slot", what);
  if (status & kErrDuplicate) return mfail(g, NOSA_ERR_VALUE, "%s: key already mapped", what);
  return mfail(g, NOSA_ERR_STATE, "%s: status %d", what, status);
}

extern "C" int nosa_mgr_create(int heads, int fast_blocks, int slow_blocks, int n_b, int d_head, int element_width,
                               int store_payload, int device, NosaMgr** out) {
  if (!out) return NOSA_ERR_VALUE;
  *out = nullptr;
  if (heads <= 0 || fast_blocks < 0 || slow_blocks < 0 || n_b <= 0 || d_head <= 0 ||
      (element_width != 2 && element_width != 4))
    return NOSA_ERR_VALUE;
  auto* g = new NosaMgr();
  g->device = device;
  g->n_b = n_b;
  g->d_head = d_head;
  g->elem = element_width;
  cudaSetDevice(device);
  Mgr& m = g->m;
  m.H = heads;
  m.F = fast_blocks;
  m.S = slow_blocks;
  m.ids = fast_blocks + slow_blocks;
  m.bpb = 2LL * n_b * d_head * element_width;
  const size_t HI = (size_t)heads * m.ids;
  int rc = NOSA_OK;
  auto step = [&](int r) { if (!rc) rc = r; };
  step(malloc_zero(g, &m.tier, HI, 0xff));
  step(malloc_zero(g, &m.slot, HI));
  step(malloc_zero(g, &m.last, HI));
  step(malloc_zero(g, &m.kb, HI));
  step(malloc_zero(g, &m.fast_id, (size_t)heads * m.F, 0xff));
  step(malloc_zero(g, &m.slow_id, (size_t)heads * m.S, 0xff));
  step(malloc_zero(g, &m.fast_free, (size_t)heads * m.F));
  step(malloc_zero(g, &m.slow_free, (size_t)heads * m.S));
  step(malloc_zero(g, &m.tops, (size_t)heads * 2));
  step(malloc_zero(g, &m.clock, 1));
  step(malloc_zero(g, &m.status, 1));
  g->io_ints = 16 + 8 * (size_t)(m.F + m.S);
  step(malloc_zero(g, &m.io, g->io_ints));
  if (rc) {
    nosa_mgr_destroy(g);
    return rc;
  }
  if (cudaHostAlloc(reinterpret_cast<void**>(&g->h_io), g->io_ints * sizeof(int), cudaHostAllocDefault) != cudaSuccess ||
      cudaStreamCreateWithFlags(&g->st, cudaStreamNonBlocking) != cudaSuccess) {
    nosa_mgr_destroy(g);
    return NOSA_ERR_CUDA;
  }
  // free lists initialised [N-1, ..., 0]: pops return 0, 1, 2, ... (kv_manager.py:147-150)
  std::vector<int> init(std::max(m.F, m.S)), tops(2 * heads);
  for (int h = 0; h < heads; ++h) {
    for (int i = 0; i < m.F; ++i) init[i] = m.F - 1 - i;
    if (m.F) cudaMemcpy(m.fast_free + (size_t)h * m.F, init.data(), m.F * sizeof(int), cudaMemcpyHostToDevice);
    for (int i = 0; i < m.S; ++i) init[i] = m.S - 1 - i;
    if (m.S) cudaMemcpy(m.slow_free + (size_t)h * m.S, init.data(), m.S * sizeof(int), cudaMemcpyHostToDevice);
    tops[2 * h] = m.F;
    tops[2 * h + 1] = m.S;
  }
  cudaMemcpy(m.tops, tops.data(), tops.size() * sizeof(int), cudaMemcpyHostToDevice);
  if (store_payload) {
    const size_t fb = (size_t)m.F * heads * m.bpb, sb = (size_t)m.S * heads * m.bpb;
    if (malloc_zero(g, &m.pay_fast, std::max<size_t>(fb, 16)) ||
        cudaHostAlloc(reinterpret_cast<void**>(&g->host_pay), std::max<size_t>(sb, 16), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(reinterpret_cast<void**>(&m.pay_slow), g->host_pay, 0) != cudaSuccess) {
      nosa_mgr_destroy(g);
      return NOSA_ERR_CUDA;
    }
    memset(g->host_pay, 0, std::max<size_t>(sb, 16));
  }
  if (cudaDeviceSynchronize() != cudaSuccess) {
    nosa_mgr_destroy(g);
    return NOSA_ERR_CUDA;
  }
  *out = g;
  return NOSA_OK;
}

extern "C" void nosa_mgr_destroy(NosaMgr* g) {
  if (!g) return;
  cudaSetDevice(g->device);
  cudaDeviceSynchronize();
  for (void* p : g->allocs) cudaFree(p);
  if (g->host_pay) cudaFreeHost(g->host_pay);
  if (g->h_io) cudaFreeHost(g->h_io);
  if (g->st) cudaStreamDestroy(g->st);
  delete g;
}

extern "C" const char* nosa_mgr_last_error(const NosaMgr* g) { return g ? g->err.c_str() : ""; }

static int check_head_id(NosaMgr* g, int head, int id) {
  if (!g) return NOSA_ERR_VALUE;
  if (head < 0 || head >= g->m.H) return mfail(g, NOSA_ERR_VALUE, "head %d out of range", head);
  if (id < 0 || id >= g->m.ids) return mfail(g, NOSA_ERR_VALUE, "key id %d out of range", id);
  cudaSetDevice(g->device);
  return NOSA_OK;
}

extern "C" int nosa_mgr_allocate(NosaMgr* g, int tier, int head, int id, int batch, int block, int32_t* slot) {
  if (int rc = check_head_id(g, head, id)) return rc;
  if (tier != 0 && tier != 1) return mfail(g, NOSA_ERR_VALUE, "tier must be 0 (fast) or 1 (slow)");
  mgr_allocate_kernel<<<1, 1, 0, g->st>>>(g->m, head, id, tier, batch, block);
  if (int rc = finish(g, "allocate")) return rc;
  MGR_TRY(g, cudaMemcpyAsync(g->h_io, g->m.io, sizeof(int), cudaMemcpyDeviceToHost, g->st));
  MGR_TRY(g, cudaStreamSynchronize(g->st));
  if (slot) *slot = g->h_io[0];
  return NOSA_OK;
}

extern "C" int nosa_mgr_free(NosaMgr* g, int head, int id) {
  if (int rc = check_head_id(g, head, id)) return rc;
  mgr_free_kernel<<<1, 1, 0, g->st>>>(g->m, head, id);
  return finish(g, "free_block");
}

extern "C" int nosa_mgr_plan(NosaMgr* g, int head, int batch, const int32_t* ids, int n, int32_t* fetch,
                             int32_t* n_fetch, int32_t* evict, int32_t* n_evict, int32_t* hits) {
  if (!g || n < 0 || (n && !ids) || !fetch || !n_fetch || !evict || !n_evict || !hits) return NOSA_ERR_VALUE;
  if (head < 0 || head >= g->m.H) return mfail(g, NOSA_ERR_VALUE, "head %d out of range", head);
  cudaSetDevice(g->device);
  if (n > g->m.F) n = g->m.F + 1;  // CapacityExceeded either way (checked before any key)
  g->h_io[0] = n;
  std::copy(ids, ids + n, g->h_io + 1);
  MGR_TRY(g, cudaMemcpyAsync(g->m.io, g->h_io, (n + 1) * sizeof(int), cudaMemcpyHostToDevice, g->st));
  mgr_plan_kernel<<<1, kThreads, 0, g->st>>>(g->m, head, batch, 0);
  if (int rc = finish(g, "plan_transfers")) return rc;
  const size_t base = 1 + n;
  MGR_TRY(g, cudaMemcpyAsync(g->h_io + base, g->m.io + base, 3 * sizeof(int), cudaMemcpyDeviceToHost, g->st));
  MGR_TRY(g, cudaStreamSynchronize(g->st));
  const int nf = g->h_io[base], ne = g->h_io[base + 1];
  if (nf + ne)
    MGR_TRY(g, cudaMemcpyAsync(g->h_io + base + 3, g->m.io + base + 3, (nf + ne) * sizeof(int), cudaMemcpyDeviceToHost,
                               g->st));
  MGR_TRY(g, cudaStreamSynchronize(g->st));
  *n_fetch = nf;
  *n_evict = ne;
  *hits = g->h_io[base + 2];
  std::copy(g->h_io + base + 3, g->h_io + base + 3 + nf, fetch);
  std::copy(g->h_io + base + 3 + nf, g->h_io + base + 3 + nf + ne, evict);
  return NOSA_OK;
}

extern "C" int nosa_mgr_apply(NosaMgr* g, int head, const int32_t* evict, int n_evict, const int32_t* fetch,
                              int n_fetch, int copy_payload, int32_t* moves) {
  if (!g || n_evict < 0 || n_fetch < 0 || (n_evict && !evict) || (n_fetch && !fetch)) return NOSA_ERR_VALUE;
  if (head < 0 || head >= g->m.H) return mfail(g, NOSA_ERR_VALUE, "head %d out of range", head);
  const int nm = n_evict + n_fetch;
  if ((size_t)(2 + 3 * nm) > g->io_ints - 1) return mfail(g, NOSA_ERR_VALUE, "plan larger than the manager");
  cudaSetDevice(g->device);
  g->h_io[0] = n_evict;
  g->h_io[1] = n_fetch;
  std::copy(evict, evict + n_evict, g->h_io + 2);
  std::copy(fetch, fetch + n_fetch, g->h_io + 2 + n_evict);
  MGR_TRY(g, cudaMemcpyAsync(g->m.io, g->h_io, (2 + nm) * sizeof(int), cudaMemcpyHostToDevice, g->st));
  mgr_apply_kernel<<<1, kThreads, 0, g->st>>>(g->m, head, copy_payload);
  if (int rc = finish(g, "apply_transfers")) return rc;
  if (moves && nm) {
    MGR_TRY(g, cudaMemcpyAsync(moves, g->m.io + 2 + nm, 2 * nm * sizeof(int), cudaMemcpyDeviceToHost, g->st));
    MGR_TRY(g, cudaStreamSynchronize(g->st));
  }
  return NOSA_OK;
}

extern "C" int nosa_mgr_lookup(NosaMgr* g, int head, int id, int32_t* tier, int32_t* slot) {
  if (int rc = check_head_id(g, head, id)) return rc;
  int8_t t = -1;
  int s = -1;
  MGR_TRY(g, cudaMemcpyAsync(&t, g->m.tier + (size_t)head * g->m.ids + id, 1, cudaMemcpyDeviceToHost, g->st));
  MGR_TRY(g, cudaMemcpyAsync(&s, g->m.slot + (size_t)head * g->m.ids + id, sizeof(int), cudaMemcpyDeviceToHost, g->st));
  MGR_TRY(g, cudaStreamSynchronize(g->st));
  if (tier) *tier = t;
  if (slot) *slot = t >= 0 ? s : -1;
  return NOSA_OK;
}

extern "C" int nosa_mgr_tables(NosaMgr* g, int head, int8_t* tier, int32_t* slot) {
  if (!g || head < 0 || head >= g->m.H || !tier || !slot) return NOSA_ERR_VALUE;
  cudaSetDevice(g->device);
  MGR_TRY(g, cudaMemcpyAsync(tier, g->m.tier + (size_t)head * g->m.ids, g->m.ids, cudaMemcpyDeviceToHost, g->st));
  MGR_TRY(g, cudaMemcpyAsync(slot, g->m.slot + (size_t)head * g->m.ids, g->m.ids * sizeof(int), cudaMemcpyDeviceToHost, g->st));
  MGR_TRY(g, cudaStreamSynchronize(g->st));
  return NOSA_OK;
}

extern "C" int nosa_mgr_audit(NosaMgr* g, int32_t* bad) {
  if (!g || !bad) return NOSA_ERR_VALUE;
  cudaSetDevice(g->device);
  MGR_TRY(g, cudaMemsetAsync(g->m.io, 0, sizeof(int), g->st));
  mgr_audit_kernel<<<g->m.H, 256, 0, g->st>>>(g->m, g->m.io);
  MGR_TRY(g, cudaGetLastError());
  MGR_TRY(g, cudaMemcpyAsync(bad, g->m.io, sizeof(int), cudaMemcpyDeviceToHost, g->st));
  MGR_TRY(g, cudaStreamSynchronize(g->st));
  return NOSA_OK;
}

extern "C" int nosa_mgr_block(NosaMgr* g, int head, int id, void* data, int write) {
  if (int rc = check_head_id(g, head, id)) return rc;
  if (!g->m.pay_fast) return mfail(g, NOSA_ERR_STATE, "manager was created without payload storage");
  if (!data) return NOSA_ERR_VALUE;
  int32_t tier = -1, slot = -1;
  if (int rc = nosa_mgr_lookup(g, head, id, &tier, &slot)) return rc;
  if (tier < 0) return mfail(g, NOSA_ERR_UNKNOWN_KEY, "key is not mapped");
  const size_t off = ((size_t)slot * g->m.H + head) * g->m.bpb;
  if (tier == 1) {  // SLOW: pinned host memory
    char* p = g->host_pay + off;
    if (write) memcpy(p, data, g->m.bpb); else memcpy(data, p, g->m.bpb);
    return NOSA_OK;
  }
  char* p = g->m.pay_fast + off;
  MGR_TRY(g, write ? cudaMemcpy(p, data, g->m.bpb, cudaMemcpyHostToDevice) : cudaMemcpy(data, p, g->m.bpb, cudaMemcpyDeviceToHost));
  return NOSA_OK;
}

extern "C" int nosa_mgr_free_lists(NosaMgr* g, int head, int32_t* fast, int32_t* n_fast, int32_t* slow, int32_t* n_slow) {
  if (!g || head < 0 || head >= g->m.H || !fast || !n_fast || !slow || !n_slow) return NOSA_ERR_VALUE;
  cudaSetDevice(g->device);
  int tops[2];
  MGR_TRY(g, cudaMemcpy(tops, g->m.tops + 2 * head, sizeof(tops), cudaMemcpyDeviceToHost));
  MGR_TRY(g, cudaMemcpy(fast, g->m.fast_free + (size_t)head * g->m.F, tops[0] * sizeof(int), cudaMemcpyDeviceToHost));
  MGR_TRY(g, cudaMemcpy(slow, g->m.slow_free + (size_t)head * g->m.S, tops[1] * sizeof(int), cudaMemcpyDeviceToHost));
  *n_fast = tops[0];
  *n_slow = tops[1];
  return NOSA_OK;
}

extern "C" int nosa_mgr_plan_policy(NosaMgr* g, int head, int batch, const int32_t* ids, int n, int32_t* fetch,
                                    int32_t* n_fetch, int32_t* shortfall, int32_t* candidates, int32_t* n_cand,
                                    int32_t* hits) {
  if (!g || n < 0 || (n && !ids) || !fetch || !n_fetch || !shortfall || !candidates || !n_cand || !hits)
    return NOSA_ERR_VALUE;
  if (head < 0 || head >= g->m.H) return mfail(g, NOSA_ERR_VALUE, "head %d out of range", head);
  cudaSetDevice(g->device);
  if (n > g->m.F) n = g->m.F + 1;
  g->h_io[0] = n;
  std::copy(ids, ids + n, g->h_io + 1);
  MGR_TRY(g, cudaMemcpyAsync(g->m.io, g->h_io, (n + 1) * sizeof(int), cudaMemcpyHostToDevice, g->st));
  mgr_plan_kernel<<<1, kThreads, 0, g->st>>>(g->m, head, batch, 1);
  if (int rc = finish(g, "plan_transfers")) return rc;
  const size_t base = 1 + n;
  // fetch ids, then (when evictions are needed) the candidate count and ids: at most 3 + F + 1 + F
  const size_t span = std::min<size_t>(4 + 2 * (size_t)g->m.F, g->io_ints - 1 - base);
  MGR_TRY(g, cudaMemcpyAsync(g->h_io + base, g->m.io + base, span * sizeof(int), cudaMemcpyDeviceToHost, g->st));
  MGR_TRY(g, cudaStreamSynchronize(g->st));
  const int nf = g->h_io[base], sf = g->h_io[base + 1];
  *n_fetch = nf;
  *shortfall = sf;
  *hits = g->h_io[base + 2];
  std::copy(g->h_io + base + 3, g->h_io + base + 3 + nf, fetch);
  const int nc = sf > 0 ? g->h_io[base + 3 + nf] : 0;
  *n_cand = nc;
  std::copy(g->h_io + base + 4 + nf, g->h_io + base + 4 + nf + nc, candidates);
  return NOSA_OK;
}

extern "C" int nosa_mgr_recency(NosaMgr* g, int head, uint32_t* last) {
  if (!g || head < 0 || head >= g->m.H || !last) return NOSA_ERR_VALUE;
  cudaSetDevice(g->device);
  MGR_TRY(g, cudaMemcpyAsync(last, g->m.last + (size_t)head * g->m.ids, g->m.ids * sizeof(unsigned),
                             cudaMemcpyDeviceToHost, g->st));
  MGR_TRY(g, cudaStreamSynchronize(g->st));
  return NOSA_OK;
}
