// nosa_attend.cu — K4 block-sparse biased decode attention + K5 append.
//
// Restates, per (sequence, kv head), the attention half of DecodeEngine.step
// (decode.py:178-185): for each query head of the GQA group, softmax over the attended
// tokens of  q.k_j + beta_j  (unscaled logits, attention.py:180) with beta_j the block-mean
// eviction score of token j's block (decode.py:180-181, 192-194; bias_logit_offsets
// attention.py:149-164), then w.V.  Masked tokens (outside Gamma(t)) contribute exactly zero,
// so only the required blocks are read; the partial tail block is clipped at t
// (selection.py:104-107).  After attention the new token is appended (decode.py:187-189) with
// its importance score (importance_scores, attention.py:121-146).
//
// Work decomposition: each (b, h) required list is cut into chunks of kChunk blocks (a fixed
// split, so results do not depend on the grid, the batch composition or the GPU count).
// bf16 kernel, one persistent CTA per SM, warp-specialised:
//   scheduler warp  claims chunks from a per-layer counter and stages their metadata (slot,
//                   token count, block bias) in a shared-memory queue;
//   copy warp       streams each 32 KiB K|V block HBM -> shared memory with one 1-D TMA bulk
//                   copy (cp.async.bulk, SASS UBLKCP) into a ring of stages (mbarrier
//                   full/empty pairs), plus the chunk's query rows;
//   4 consumer warps split every block by keys (16 keys each) and run QK^T and PV on the
//                   tensor cores with keys on M and the GQA group's queries on N
//                   (mma.m16n8k16, no padding for G = 8), online softmax in registers.
// At a chunk end the consumer warps combine their partials through shared memory and write
// one (m, l, O) record.  The finalize kernel (one CTA per (b, h), launched right after) merges
// the records in chunk order (log-sum-exp) and performs the append; keeping that latency-bound
// work out of the streaming kernel keeps the persistent CTAs on the HBM stream.
#include "nosa_device.cuh"

namespace nosa {

constexpr float kLog2e = 1.4426950408889634f;
constexpr int kBarConsumers = 1;  // named barrier id of the consumer warps

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ int find_bh(const int* cbase, int BH, int c) {
  int lo = 0, hi = BH;  // largest bh with cbase[bh] <= c
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (cbase[mid] <= c) lo = mid; else hi = mid;
  }
  return lo;
}

// block-level exclusive scan of ceil(n_req/chunk) over the BH (b, h) entries into cbase:
// per-thread sums of a contiguous range, a shuffle scan inside each warp, then the warp totals
// (tmp[0..nwarps)) scanned by every thread.  Two barriers, no serial loop.
__device__ void chunk_scan(const Dev& dv, int layer, int* cbase, int* tmp, int units = -1) {
  const int BH = units < 0 ? dv.B * dv.H : units;  // units of layers [layer, ...) are contiguous
  const int nt = blockDim.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = nt >> 5;
  const int per = (BH + nt - 1) / nt;
  const int lo = min(BH, (int)threadIdx.x * per), hi = min(BH, lo + per);
  const int* nreq = dv.n_req + layer * dv.B * dv.H;
  int s = 0;
  for (int i = lo; i < hi; ++i) s += (nreq[i] + dv.chunk - 1) / dv.chunk;
  int incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) tmp[warp] = incl;
  __syncthreads();
  int base = 0, total = 0;
  for (int w = 0; w < nwarps; ++w) {
    const int v = tmp[w];
    base += w < warp ? v : 0;
    total += v;
  }
  int acc = base + incl - s;
  for (int i = lo; i < hi; ++i) {
    cbase[i] = acc;
    acc += (nreq[i] + dv.chunk - 1) / dv.chunk;
  }
  if (threadIdx.x == 0) cbase[BH] = total;
  __syncthreads();
}

// beta of one block: block-mean score, the tail block over its t - blk*n_b live tokens
__device__ __forceinline__ float block_beta(const Dev& dv, int lbh, int blk, int t) {
  const int n_b = dv.n_b;
  double m;
  if ((blk + 1) * n_b <= t) {
    m = dv.se[(size_t)lbh * dv.NB + blk];
  } else {
    m = dv.tail_se[lbh] / (double)(t - blk * n_b);
  }
  if (dv.variant == 1) return 0.0f;
  if (dv.variant == 2) return (float)log(m);
  return (float)m;
}

// ---------------------------------------------------------------- finalize (merge + append)
// One CTA (kFinThreads threads) per (b, h).  The kernel is latency-bound, so it is organised
// around dependent global round trips: every operand that does not depend on another load
// (the new K/V row, the eviction-head operands, the tail sums, the cache length) is loaded up
// front, the split-K records are merged with an online log-sum-exp in record order (batches of
// 8 records in flight per thread), and only the slot lookup of the tail block waits on t.
constexpr int kFinThreads = 256;
constexpr int kFinMaxRows = 16;  // eviction-head rows per thread (D / (kFinThreads / n_ev))

template <typename T>
__device__ void finalize_bh(const Dev& dv, int layer, int bh, const T* __restrict__ kn,
                            const T* __restrict__ vn, float* __restrict__ out, float* wsm, double* zsm) {
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int b = bh / dv.H, h = bh % dv.H;
  const int lbh = (layer * dv.B + b) * dv.H + h;
  const int D = dv.D, G = dv.G, n_b = dv.n_b, n_ev = dv.n_ev, elem = dv.elem;
  const T* kr = kn + ((size_t)b * dv.H + h) * D;
  const T* vr = vn + ((size_t)b * dv.H + h) * D;

  // ---- (0) independent loads: t, the record count, the new row's 16-byte chunks, eviction-head
  //          operands, tail sums
  const int t = __ldcg(dv.t + lbh);
  const int n_req = __ldcg(dv.n_req + (size_t)layer * dv.B * dv.H + bh);
  const int cpr = D * elem / 16;  // 16-byte chunks per row
  int4 rowv = make_int4(0, 0, 0, 0);
  if (tid < 2 * cpr) rowv = reinterpret_cast<const int4*>(tid < cpr ? (const void*)kr : (const void*)vr)[tid % cpr];
  // importance score s = silu(v . W1) . W2 (attention.py:121-146): thread -> (column j, row group)
  const int groups = nthr / n_ev, rpg = (D + groups - 1) / groups;
  const bool ev_fast = groups > 0 && rpg <= kFinMaxRows;
  const int j_ev = tid % max(n_ev, 1), grp = tid / max(n_ev, 1);
  double part = 0.0;
  if (ev_fast && grp < groups) {
    double vv[kFinMaxRows], ww[kFinMaxRows];
#pragma unroll
    for (int u = 0; u < kFinMaxRows; ++u) {
      const int i = grp * rpg + u;
      const bool ok = u < rpg && i < D;
      vv[u] = ok ? to_f64(vr[i]) : 0.0;
      ww[u] = ok ? __ldg(dv.w1 + (size_t)i * n_ev + j_ev) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kFinMaxRows; ++u) part = fma(vv[u], ww[u], part);
  }
  double tks = 0.0, kv = 0.0;
  if (tid < D) {
    tks = __ldcg(dv.tail_ksum + (size_t)lbh * D + tid);
    kv = to_f64(kr[tid]);
  }
  const double tse = __ldcg(dv.tail_se + lbh);

  const int nc = (n_req + dv.chunk - 1) / dv.chunk;
  if (nc == 0) return;  // the plan failed for this manager (CapacityExceeded): no step

  // ---- (1) merge the split-K records in record order (deterministic), thread -> (query, 4 dims)
  {
    const int D4 = D / 4;
    const float2* ml = part_ml_of(dv, layer) + (size_t)bh * dv.max_chunks * G;
    const float4* po = reinterpret_cast<const float4*>(part_o_of(dv, layer) + (size_t)bh * dv.max_chunks * G * D);
    for (int x = tid; x < G * D4; x += nthr) {
      const int q = x / D4, d4 = x - q * D4;
      float M = -INFINITY, L = 0.0f;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int c0 = 0; c0 < nc; c0 += 8) {
        float2 m8[8];
        float4 o8[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int c = c0 + u;
          m8[u] = c < nc ? __ldcg(ml + (size_t)c * G + q) : make_float2(-INFINITY, 0.f);
          o8[u] = c < nc ? __ldcg(po + ((size_t)c * G + q) * D4 + d4) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (m8[u].x == -INFINITY) continue;  // a record over no live key
          const float Mn = fmaxf(M, m8[u].x);
          const float a = expf(M - Mn), e = expf(m8[u].x - Mn);
          L = fmaf(L, a, m8[u].y * e);
          acc.x = fmaf(acc.x, a, o8[u].x * e);
          acc.y = fmaf(acc.y, a, o8[u].y * e);
          acc.z = fmaf(acc.z, a, o8[u].z * e);
          acc.w = fmaf(acc.w, a, o8[u].w * e);
          M = Mn;
        }
      }
      const float inv = 1.0f / L;
      reinterpret_cast<float4*>(out + ((size_t)b * dv.Hq + h * G + q) * D)[d4] =
          make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
    }
  }

  // ---- (2) append the new token (decode.py:187-189, HeadState.append decode.py:65-71)
  if (t >= dv.NB * n_b) {  // head cache full (HeadState capacity): refuse the append, flag it
    if (tid == 0) atomicOr(dv.err, 8u);  // NOSA_FLAG_FULL
    return;
  }
  const int blk = t / n_b, r = t - blk * n_b;
  const int plane = n_b * D * elem;
  char* hblk = dv.host + ((size_t)lbh * dv.NB + blk) * dv.bpb;
  if (tid < 2 * cpr) {
    const int sl = __ldcg(dv.slot_of + (size_t)lbh * dv.NB + blk);
    const long long slot = sl < 0 ? -1 : (dv.shared ? shared_rel(dv, b, sl) : sl);  // relative to this row
    const int which = tid / cpr, ch = tid - which * cpr;
    const int off = which * plane + r * D * elem + ((ch ^ (r & 7)) << 4);
    *reinterpret_cast<int4*>(hblk + off) = rowv;
    if (sl >= 0) *reinterpret_cast<int4*>(dv.pool + ((long long)lbh * dv.C + slot) * dv.bpb + off) = rowv;
    if (r == 0) reinterpret_cast<int4*>(dv.newrow + (size_t)lbh * 2 * D * elem)[tid] = rowv;  // see gather_kernel
  }
  // (A new block's unwritten rows need no zero-fill in the slow tier: prefill zero-pads every
  // block past t, appended rows are real data, and rows past the live count are masked out of
  // attention.  Filling them cost 32 KiB of posted host writes per unit at each block boundary:
  // 235 MB in one step when a whole cfg 3 batch crosses a boundary together.)
  // running key sums of the tail block -> K_c of a completed block (compress_blocks)
  if (tid < D) {
    const double acc = (r == 0) ? kv : tks + kv;
    if (r == n_b - 1) {
      dv.kc[((size_t)lbh * dv.NB + blk) * D + tid] = acc / (double)n_b;
      dv.tail_ksum[(size_t)lbh * D + tid] = 0.0;
    } else {
      dv.tail_ksum[(size_t)lbh * D + tid] = acc;
    }
  }
  // eviction-head column sums: row-group partials -> silu per column
  double* red = reinterpret_cast<double*>(wsm);  // [nthr]
  if (ev_fast) {
    red[tid] = part;
    __syncthreads();
    if (tid < n_ev) {
      double zc = 0.0;
      for (int g2 = 0; g2 < groups; ++g2) zc += red[g2 * n_ev + tid];
      zsm[tid] = silu64(zc);
    }
  } else {  // wide heads: one warp per column
    const int lane = tid & 31, warp = tid >> 5, nwarps = nthr >> 5;
    for (int j = warp; j < n_ev; j += nwarps) {
      double p2 = 0.0;
      for (int i = lane; i < D; i += 32) p2 = fma(to_f64(vr[i]), dv.w1[(size_t)i * n_ev + j], p2);
#pragma unroll
      for (int o = 16; o; o >>= 1) p2 += __shfl_xor_sync(0xffffffffu, p2, o);
      if (lane == 0) zsm[j] = silu64(p2);
    }
  }
  __syncthreads();
  if (tid == 0) {
    double z = 0.0;
    for (int j = 0; j < n_ev; ++j) z = fma(zsm[j], dv.w2[j], z);
    const double sc = dv.variant == 2 ? exp(z) : z;
    const double acc = (r == 0) ? sc : tse + sc;
    if (r == n_b - 1) {
      dv.se[(size_t)lbh * dv.NB + blk] = acc / (double)n_b;
      dv.tail_se[lbh] = 0.0;
    } else {
      dv.tail_se[lbh] = acc;
    }
    dv.t[lbh] = t + 1;
  }
  // No system fence: within a run the slow copy of a just-written row is never read back (a
  // block born by this append is rebuilt from dv.newrow); later readers follow a host sync.
}

// ---------------------------------------------------------------- bf16 tensor-core kernel
template <int NBK, int DH, int NQT>
struct BF {
  static constexpr int BPB = 2 * NBK * DH * 2;
  static constexpr int PLANE = NBK * DH * 2;
  static constexpr int NCW = NBK >= 64 ? 4 : NBK / 16;  // consumer warps
  static constexpr int KPW = NBK / NCW;                 // keys per consumer warp
  static constexpr int MTK = KPW / 16;                  // key m-tiles per warp
  static constexpr int MTD = DH / 16;                   // head-dim m-tiles (PV)
  static constexpr int KS = DH / 16;                    // k-steps (QK)
  static constexpr int QMAX = 8 * NQT;                  // queries per (b, h), padded to n-tiles
  static constexpr int QROW = DH * 2 + 16;               // padded query row: fragment loads hit 8 banks
  static constexpr int QSLOT = QMAX * QROW;
  static constexpr int CLD = DH + 4;                     // padded f32 row of the warp-combine buffer
  static constexpr int COMB = NCW * QMAX * CLD * 4 + NCW * QMAX * 8;
  static constexpr int NSR = (200 * 1024 - COMB) / (BPB + QSLOT);
  static constexpr int NS = NSR > 8 ? 8 : (NSR < 2 ? 2 : NSR);  // ring stages
  static constexpr int NQ = 3;                                  // chunk-metadata queue depth
  static constexpr int THREADS = (NCW + 2) * 32;                // + copy warp + scheduler warp
  static constexpr int WARP_COPY = NCW, WARP_SCHED = NCW + 1;
};

struct ItemInfo {
  int bh, ci, flags, count;
  float beta;
  int nc, pad0, pad1;
};
enum { IF_FIRST = 1, IF_LAST = 2, IF_END = 4 };

struct ChunkMeta {
  int bh, ci, n, nc;
  int slot[kChunk];
  int count[kChunk];
  float beta[kChunk];
};

template <int NBK, int DH, int NQT>
__host__ __device__ constexpr size_t bf_smem_fixed() {
  using T = BF<NBK, DH, NQT>;
  return (size_t)T::NS * T::BPB + (size_t)T::NS * T::QSLOT + T::COMB + 2 * T::NS * 8 + 2 * T::NQ * 8 +
         T::NS * sizeof(ItemInfo) + T::NQ * sizeof(ChunkMeta) + T::THREADS * 4 + 64;
}

template <int NBK, int DH, int NQT>
__global__ void __launch_bounds__(BF<NBK, DH, NQT>::THREADS, 1)
    attend_bf16_kernel(Dev dv, int layer, int nl, const __nv_bfloat16* __restrict__ q, size_t q_layer_stride) {
  // layers [layer, layer + nl) in one persistent launch: work unit u = (layer - layer0) * B*H + bh,
  // so lbh = layer0 * B*H + u and the units of all layers form one contiguous list
  using T = BF<NBK, DH, NQT>;
  extern __shared__ __align__(128) char smem_raw[];
  const int BHL = dv.B * dv.H;
  const int BH = nl * BHL;
  const int G = dv.G;
  char* p = smem_raw;
  char* stages = p;                                   p += (size_t)T::NS * T::BPB;
  char* qslots = p;                                   p += (size_t)T::NS * T::QSLOT;
  float* comb_o = reinterpret_cast<float*>(p);        p += (size_t)T::NCW * T::QMAX * T::CLD * 4;
  float2* comb_ml = reinterpret_cast<float2*>(p);     p += (size_t)T::NCW * T::QMAX * 8;
  uint64_t* full = reinterpret_cast<uint64_t*>(p);    p += T::NS * 8;
  uint64_t* empty = reinterpret_cast<uint64_t*>(p);   p += T::NS * 8;
  uint64_t* mq_full = reinterpret_cast<uint64_t*>(p); p += T::NQ * 8;
  uint64_t* mq_empty = reinterpret_cast<uint64_t*>(p); p += T::NQ * 8;
  ItemInfo* info = reinterpret_cast<ItemInfo*>(p);    p += T::NS * sizeof(ItemInfo);
  ChunkMeta* meta = reinterpret_cast<ChunkMeta*>(p);  p += T::NQ * sizeof(ChunkMeta);
  int* tmp = reinterpret_cast<int*>(p);               p += T::THREADS * 4;
  int* flag = reinterpret_cast<int*>(p);              p += 64;
  int* cbase = reinterpret_cast<int*>(p);             p += (size_t)(BH + 1) * 4;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned long long t_start = dv.ktime ? globaltimer_ns() : 0ull;
  if (tid == 0) {
    for (int s = 0; s < T::NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], T::NCW);
    }
    for (int s = 0; s < T::NQ; ++s) {
      mbar_init(&mq_full[s], 1);
      mbar_init(&mq_empty[s], 1);
    }
    fence_mbar_init();
  }
  if (G < T::QMAX)  // query rows past the group stay zero (only G rows are ever copied in)
    for (int x = tid; x < T::NS * T::QSLOT / 16; x += blockDim.x) reinterpret_cast<int4*>(qslots)[x] = make_int4(0, 0, 0, 0);
  chunk_scan(dv, layer, cbase, tmp, BH);  // also publishes the barrier inits (__syncthreads)
  const int total = cbase[BH];

  if (warp == T::WARP_SCHED) {
    // ------------------------------------------------------------ scheduler warp
    for (int qs = 0;; ++qs) {
      // the first work item is static (item = CTA index), later ones are claimed dynamically
      int c = blockIdx.x;
      if (qs > 0) {
        if (lane == 0) c = gridDim.x + atomicAdd(dv.cnt + kCntStride * layer + 1, 1);
        c = __shfl_sync(0xffffffffu, c, 0);
      }
      const int slot = qs % T::NQ;
      mbar_wait(&mq_empty[slot], ((qs / T::NQ) & 1) ^ 1);
      ChunkMeta& m = meta[slot];
      if (c >= total) {
        if (lane == 0) {
          m.n = -1;
          mbar_arrive(&mq_full[slot]);
        }
        break;
      }
      const int bh = find_bh(cbase, BH, c);
      const int lbh = layer * BHL + bh;
      const int ci = c - cbase[bh];
      const int nreq = dv.n_req[lbh];
      const int t = dv.t[lbh];
      const int i0 = ci * dv.chunk;
      const int n = min(dv.chunk, nreq - i0);
      if (lane < n) {
        const int blk = dv.req[(size_t)lbh * dv.C + i0 + lane];
        m.slot[lane] = dv.req_slot[(size_t)lbh * dv.C + i0 + lane];
        m.count[lane] = min(NBK, t - blk * NBK);
        m.beta[lane] = block_beta(dv, lbh, blk, t);
      }
      if (lane == 0) {
        m.bh = bh;
        m.ci = ci;
        m.n = n;
        m.nc = (nreq + dv.chunk - 1) / dv.chunk;
      }
      __threadfence_block();
      __syncwarp();
      if (lane == 0) mbar_arrive(&mq_full[slot]);
    }
  } else if (warp == T::WARP_COPY) {
    // ------------------------------------------------------------ copy warp (TMA producer)
    int seq = 0;
    for (int qs = 0;; ++qs) {
      const int slot = qs % T::NQ;
      mbar_wait(&mq_full[slot], (qs / T::NQ) & 1);
      const ChunkMeta& m = meta[slot];
      const int n = m.n;
      if (n < 0) break;
      const int bh = m.bh, ci = m.ci, nc = m.nc;
      const int lbh = layer * BHL + bh;
      const int bhl = bh % BHL, b = bhl / dv.H, h = bhl - b * dv.H;
      const __nv_bfloat16* ql = q + (size_t)(bh / BHL) * q_layer_stride;
      for (int i = 0; i < n; ++i, ++seq) {
        const int s = seq % T::NS;
        mbar_wait(&empty[s], ((seq / T::NS) & 1) ^ 1);
        if (lane == 0) {
          ItemInfo& it = info[s];
          it.bh = bh;
          it.ci = ci;
          it.flags = (i == 0 ? IF_FIRST : 0) | (i == n - 1 ? IF_LAST : 0);
          it.count = m.count[i];
          it.beta = m.beta[i];
          it.nc = nc;
        }
        __threadfence_block();
        __syncwarp();
        if (lane == 0) {
          fence_proxy_async();
          const unsigned qbytes = i == 0 ? (unsigned)(G * DH * 2) : 0u;  // the chunk's query rows
          mbar_expect_tx(&full[s], T::BPB + qbytes);
          bulk_g2s(stages + (size_t)s * T::BPB, dv.pool + ((size_t)lbh * dv.C + m.slot[i]) * (size_t)T::BPB, T::BPB,
                   &full[s]);
          if (qbytes)
            for (int r = 0; r < G; ++r)  // one bulk copy per query row into the padded slot
              bulk_g2s(qslots + (size_t)s * T::QSLOT + r * T::QROW, ql + ((size_t)b * dv.Hq + h * G + r) * DH,
                       DH * 2, &full[s]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&mq_empty[slot]);
    }
    const int s = seq % T::NS;  // end-of-work marker for the consumers
    mbar_wait(&empty[s], ((seq / T::NS) & 1) ^ 1);
    if (lane == 0) {
      info[s].flags = IF_END;
      mbar_arrive(&full[s]);
    }
  } else {
    // ------------------------------------------------------------ consumer warps
    const int g = lane >> 2, tq = lane & 3;
    const int w = warp;
    unsigned qb[T::KS][NQT][2];
    float o[T::MTD][NQT][4];
    float mrun[NQT][2], lrun[NQT][2];
    for (int seq = 0;; ++seq) {
      const int s = seq % T::NS;
      mbar_wait(&full[s], (seq / T::NS) & 1);
      __syncwarp();  // lanes leave the spin-wait independently: reconverge before ldmatrix / mma (.aligned)
      const ItemInfo it = info[s];
      if (it.flags & IF_END) break;
      if (it.flags & IF_FIRST) {
        const char* qs = qslots + (size_t)s * T::QSLOT;
#pragma unroll
        for (int ks = 0; ks < T::KS; ++ks)
#pragma unroll
          for (int nq = 0; nq < NQT; ++nq) {
            const char* row = qs + (size_t)(8 * nq + g) * T::QROW;
            qb[ks][nq][0] = *reinterpret_cast<const unsigned*>(row + (16 * ks + 2 * tq) * 2);
            qb[ks][nq][1] = *reinterpret_cast<const unsigned*>(row + (16 * ks + 8 + 2 * tq) * 2);
          }
#pragma unroll
        for (int md = 0; md < T::MTD; ++md)
#pragma unroll
          for (int nq = 0; nq < NQT; ++nq) o[md][nq][0] = o[md][nq][1] = o[md][nq][2] = o[md][nq][3] = 0.0f;
#pragma unroll
        for (int nq = 0; nq < NQT; ++nq) {
          mrun[nq][0] = mrun[nq][1] = -INFINITY;
          lrun[nq][0] = lrun[nq][1] = 0.0f;
        }
      }
      const unsigned kbase = smem_u32(stages + (size_t)s * T::BPB);
      const unsigned vbase = kbase + T::PLANE;
      const int key0 = w * T::KPW;
      // ---- S^T = K Q^T : keys on M (16 per m-tile), queries on N
      float sc[T::MTK][NQT][4];
#pragma unroll
      for (int mk = 0; mk < T::MTK; ++mk)
#pragma unroll
        for (int nq = 0; nq < NQT; ++nq) sc[mk][nq][0] = sc[mk][nq][1] = sc[mk][nq][2] = sc[mk][nq][3] = 0.0f;
#pragma unroll
      for (int ks = 0; ks < T::KS; ++ks) {
#pragma unroll
        for (int mk = 0; mk < T::MTK; ++mk) {
          const int mi = lane >> 3;
          const int key = key0 + mk * 16 + (lane & 7) + 8 * (mi & 1);
          const int chunk = 2 * ks + (mi >> 1);
          unsigned a0, a1, a2, a3;
          ldsm_x4(kbase + key * (DH * 2) + ((chunk ^ (key & 7)) << 4), a0, a1, a2, a3);
#pragma unroll
          for (int nq = 0; nq < NQT; ++nq) mma_bf16(sc[mk][nq], a0, a1, a2, a3, qb[ks][nq][0], qb[ks][nq][1]);
        }
      }
      // ---- online softmax over this warp's keys, per query column
      const float beta = it.beta;
      const int count = it.count;
#pragma unroll
      for (int nq = 0; nq < NQT; ++nq) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          float mx = -INFINITY;
#pragma unroll
          for (int mk = 0; mk < T::MTK; ++mk) {
            const int klo = key0 + mk * 16 + g;
            sc[mk][nq][e] = klo < count ? sc[mk][nq][e] + beta : -INFINITY;
            sc[mk][nq][2 + e] = klo + 8 < count ? sc[mk][nq][2 + e] + beta : -INFINITY;
            mx = fmaxf(mx, fmaxf(sc[mk][nq][e], sc[mk][nq][2 + e]));
          }
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
          const float mn = fmaxf(mrun[nq][e], mx);
          const bool live = mn != -INFINITY;
          const float scale = live ? exp2f((mrun[nq][e] - mn) * kLog2e) : 1.0f;
          const float mb = live ? mn * kLog2e : 0.0f;
          float sum = 0.0f;
#pragma unroll
          for (int mk = 0; mk < T::MTK; ++mk) {
            sc[mk][nq][e] = exp2f(fmaf(sc[mk][nq][e], kLog2e, -mb));
            sc[mk][nq][2 + e] = exp2f(fmaf(sc[mk][nq][2 + e], kLog2e, -mb));
            sum += sc[mk][nq][e] + sc[mk][nq][2 + e];
          }
          lrun[nq][e] = lrun[nq][e] * scale + sum;
          mrun[nq][e] = mn;
#pragma unroll
          for (int md = 0; md < T::MTD; ++md) {
            o[md][nq][e] *= scale;
            o[md][nq][2 + e] *= scale;
          }
        }
      }
      // ---- O^T += V^T P^T : head dims on M, queries on N, this warp's keys on K
      const int src0 = 8 * tq + (g >> 1);
      const unsigned sel = (g & 1) ? 0x7632u : 0x5410u;
#pragma unroll
      for (int mk = 0; mk < T::MTK; ++mk) {
        unsigned pb[NQT][2];
#pragma unroll
        for (int nq = 0; nq < NQT; ++nq) {
          const unsigned x01 = pack_bf16(sc[mk][nq][0], sc[mk][nq][1]);
          const unsigned x23 = pack_bf16(sc[mk][nq][2], sc[mk][nq][3]);
          const unsigned v0 = __shfl_sync(0xffffffffu, x01, src0);
          const unsigned v1 = __shfl_sync(0xffffffffu, x01, src0 + 4);
          const unsigned v2 = __shfl_sync(0xffffffffu, x23, src0);
          const unsigned v3 = __shfl_sync(0xffffffffu, x23, src0 + 4);
          pb[nq][0] = __byte_perm(v0, v1, sel);
          pb[nq][1] = __byte_perm(v2, v3, sel);
        }
#pragma unroll
        for (int md = 0; md < T::MTD; ++md) {
          const int mi = lane >> 3;
          const int key = key0 + mk * 16 + (lane & 7) + 8 * (mi >> 1);
          const int chunk = 2 * md + (mi & 1);
          unsigned a0, a1, a2, a3;
          ldsm_x4_t(vbase + key * (DH * 2) + ((chunk ^ (key & 7)) << 4), a0, a1, a2, a3);
#pragma unroll
          for (int nq = 0; nq < NQT; ++nq) mma_bf16(o[md][nq], a0, a1, a2, a3, pb[nq][0], pb[nq][1]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);  // stage (and its query slot) may be refilled

      if (it.flags & IF_LAST) {
        // ---- chunk end: combine the consumer warps' partials, write one record
#pragma unroll
        for (int nq = 0; nq < NQT; ++nq)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            float l = lrun[nq][e];
            l += __shfl_xor_sync(0xffffffffu, l, 4);
            l += __shfl_xor_sync(0xffffffffu, l, 8);
            l += __shfl_xor_sync(0xffffffffu, l, 16);
            if (g == 0) comb_ml[w * T::QMAX + 8 * nq + 2 * tq + e] = make_float2(mrun[nq][e], l);
          }
#pragma unroll
        for (int md = 0; md < T::MTD; ++md)
#pragma unroll
          for (int nq = 0; nq < NQT; ++nq)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              float* row = comb_o + ((size_t)w * T::QMAX + 8 * nq + 2 * tq + e) * T::CLD;
              row[16 * md + g] = o[md][nq][e];
              row[16 * md + g + 8] = o[md][nq][2 + e];
            }
        named_sync(kBarConsumers, T::NCW * 32);
        const int ci = it.ci, rl = layer + it.bh / BHL;  // the record's layer and (b, h)
        const size_t pb0 = (size_t)(it.bh % BHL) * dv.max_chunks + ci;
        for (int x = tid; x < G * DH; x += T::NCW * 32) {
          const int qq = x / DH, d = x - qq * DH;
          float M = -INFINITY;
#pragma unroll
          for (int ww = 0; ww < T::NCW; ++ww) M = fmaxf(M, comb_ml[ww * T::QMAX + qq].x);
          float acc = 0.0f, L = 0.0f;
#pragma unroll
          for (int ww = 0; ww < T::NCW; ++ww) {
            const float2 ml = comb_ml[ww * T::QMAX + qq];
            const float f = ml.x == -INFINITY ? 0.0f : exp2f((ml.x - M) * kLog2e);
            acc = fmaf(f, comb_o[((size_t)ww * T::QMAX + qq) * T::CLD + d], acc);
            L = fmaf(f, ml.y, L);
          }
          part_o_of(dv, rl)[(pb0 * G + qq) * DH + d] = acc;
          if (d == 0) part_ml_of(dv, rl)[pb0 * G + qq] = make_float2(M, L);
        }
        named_sync(kBarConsumers, T::NCW * 32);  // comb_* may be overwritten at the next chunk end
      }
    }
  }
  if (dv.ktime) {  // diagnostics: device-clock span of the launch (first CTA start .. last CTA end)
    __syncthreads();
    if (tid == 0) {
      atomicMin(dv.ktime + 2 * layer, t_start);
      atomicMax(dv.ktime + 2 * layer + 1, globaltimer_ns());
    }
  }
}

// ---------------------------------------------------------------- fp32 CUDA-core kernel
// Parity path for fp32 storage (tolerance 1e-5): same chunk decomposition and merge, one warp
// per CTA with a private double-buffered ring, logits and P.V in fp32 FMA with accurate expf.
template <int NBK, int DH, int NS>
__global__ void __launch_bounds__(32)
    attend_f32_kernel(Dev dv, int layer, const float* __restrict__ q, const float* __restrict__ kn,
                      const float* __restrict__ vn, float* __restrict__ out) {
  constexpr int BPB = 2 * NBK * DH * 4;
  constexpr int PLANE = NBK * DH * 4;
  constexpr int RING = NS + 2;
  constexpr int DL = DH / 32;  // dims per lane
  constexpr int GM = 16;
  extern __shared__ __align__(128) char smem_raw[];
  const int BH = dv.B * dv.H;
  char* stages = smem_raw;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + (size_t)NS * BPB);
  float* qs = reinterpret_cast<float*>(bars + NS);      // [GM][DH]
  float* ps = qs + GM * DH;                              // [GM][NBK]
  int* ring = reinterpret_cast<int*>(ps + GM * NBK);     // [RING]
  int* tmp = ring + RING;                                // [32]
  int* cbase = tmp + 32;                                 // [BH+1]
  const int lane = threadIdx.x;
  const int G = dv.G;
  if (lane == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  chunk_scan(dv, layer, cbase, tmp);
  const int total = cbase[BH];

  int ld_seq = 0, ld_chunk_n = 0, ld_bh = 0, ld_i = 0, ld_end = 0;
  bool ld_done = false;
  auto advance_loader = [&]() {
    if (ld_done) return;
    if (ld_i >= ld_end) {
      int c = 0;
      if (lane == 0) c = atomicAdd(dv.cnt + kCntStride * layer + 1, 1);
      c = __shfl_sync(0xffffffffu, c, 0);
      if (c >= total) { ld_done = true; return; }
      ld_bh = find_bh(cbase, BH, c);
      const int ci = c - cbase[ld_bh];
      ld_i = ci * dv.chunk;
      ld_end = min(ld_i + dv.chunk, dv.n_req[layer * BH + ld_bh]);
      if (lane == 0) ring[ld_chunk_n % RING] = c;
      ++ld_chunk_n;
    }
    const int lbh = layer * BH + ld_bh;
    const int slot = dv.req_slot[(size_t)lbh * dv.C + ld_i];
    const int st = ld_seq % NS;
    if (lane == 0) {
      fence_proxy_async();
      mbar_expect_tx(&bars[st], BPB);
      bulk_g2s(stages + (size_t)st * BPB, dv.pool + ((size_t)lbh * dv.C + slot) * (size_t)BPB, BPB, &bars[st]);
    }
    ++ld_i;
    ++ld_seq;
  };
  for (int s = 0; s < NS; ++s) advance_loader();
  __syncwarp();

  int cp_seq = 0, cp_chunk_n = 0, cp_bh = 0, cp_i = 0, cp_end = 0, cp_ci = 0, cp_t = 0;
  float o[GM][DL];
  float m[GM], l[GM];
  while (cp_seq < ld_seq) {
    if (cp_i >= cp_end) {
      __syncwarp();
      const int c = ring[cp_chunk_n % RING];
      ++cp_chunk_n;
      cp_bh = find_bh(cbase, BH, c);
      cp_ci = c - cbase[cp_bh];
      cp_i = cp_ci * dv.chunk;
      cp_end = min(cp_i + dv.chunk, dv.n_req[layer * BH + cp_bh]);
      cp_t = dv.t[layer * BH + cp_bh];
      const int b = cp_bh / dv.H, h = cp_bh % dv.H;
      __syncwarp();
      for (int x = lane; x < G * DH; x += 32) qs[x] = q[((size_t)b * dv.Hq + h * G) * DH + x];
#pragma unroll
      for (int gg = 0; gg < GM; ++gg) {
        m[gg] = -INFINITY;
        l[gg] = 0.0f;
#pragma unroll
        for (int x = 0; x < DL; ++x) o[gg][x] = 0.0f;
      }
      __syncwarp();
    }
    const int lbh = layer * BH + cp_bh;
    const int blk = dv.req[(size_t)lbh * dv.C + cp_i];
    const int count = min(NBK, cp_t - blk * NBK);
    const float beta = block_beta(dv, lbh, blk, cp_t);
    const int st = cp_seq % NS;
    mbar_wait(&bars[st], (cp_seq / NS) & 1);
    const char* kb = stages + (size_t)st * BPB;
    const char* vb = kb + PLANE;
    for (int key = lane; key < NBK; key += 32) {
      float acc[GM];
#pragma unroll
      for (int gg = 0; gg < GM; ++gg) acc[gg] = 0.0f;
      for (int ch = 0; ch < DH / 4; ++ch) {
        const float4 kv = *reinterpret_cast<const float4*>(kb + key * DH * 4 + ((ch ^ (key & 7)) << 4));
#pragma unroll
        for (int gg = 0; gg < GM; ++gg) {
          if (gg >= G) break;
          const float4 qv = *reinterpret_cast<const float4*>(qs + gg * DH + ch * 4);
          acc[gg] = fmaf(qv.x, kv.x, acc[gg]);
          acc[gg] = fmaf(qv.y, kv.y, acc[gg]);
          acc[gg] = fmaf(qv.z, kv.z, acc[gg]);
          acc[gg] = fmaf(qv.w, kv.w, acc[gg]);
        }
      }
#pragma unroll
      for (int gg = 0; gg < GM; ++gg) {
        if (gg >= G) break;
        ps[gg * NBK + key] = key < count ? acc[gg] + beta : -INFINITY;
      }
    }
    __syncwarp();
#pragma unroll
    for (int gg = 0; gg < GM; ++gg) {
      if (gg >= G) break;
      float mx = -INFINITY;
      for (int key = lane; key < NBK; key += 32) mx = fmaxf(mx, ps[gg * NBK + key]);
#pragma unroll
      for (int off = 16; off; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
      const float mn = fmaxf(m[gg], mx);
      const float sc = expf(m[gg] - mn);
      float sum = 0.0f;
      for (int key = lane; key < NBK; key += 32) {
        const float pr = expf(ps[gg * NBK + key] - mn);
        ps[gg * NBK + key] = pr;
        sum += pr;
      }
#pragma unroll
      for (int off = 16; off; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
      l[gg] = l[gg] * sc + sum;
      m[gg] = mn;
#pragma unroll
      for (int x = 0; x < DL; ++x) o[gg][x] *= sc;
    }
    __syncwarp();
    for (int key = 0; key < NBK; ++key) {
      float vv[DL];
#pragma unroll
      for (int x = 0; x < DL; ++x) vv[x] = *reinterpret_cast<const float*>(vb + swz_off(key, lane + 32 * x, DH, 4));
#pragma unroll
      for (int gg = 0; gg < GM; ++gg) {
        if (gg >= G) break;
        const float pr = ps[gg * NBK + key];
#pragma unroll
        for (int x = 0; x < DL; ++x) o[gg][x] = fmaf(pr, vv[x], o[gg][x]);
      }
    }
    __syncwarp();
    ++cp_seq;
    ++cp_i;
    advance_loader();
    if (cp_i >= cp_end) {
      const size_t pbase = (size_t)cp_bh * dv.max_chunks + cp_ci;
#pragma unroll
      for (int gg = 0; gg < GM; ++gg) {
        if (gg >= G) break;
        float* po = part_o_of(dv, layer) +(pbase * G + gg) * DH;
#pragma unroll
        for (int x = 0; x < DL; ++x) po[lane + 32 * x] = o[gg][x];
        if (lane == 0) part_ml_of(dv, layer)[pbase * G + gg] = make_float2(m[gg], l[gg]);
      }
      __syncwarp();
    }
  }
}

// ---------------------------------------------------------------- fp32 kernel, warp group
// fp32 storage (tolerance 1e-5): one persistent CTA per SM, the same chunk decomposition and
// (m, l, O) records as the bf16 kernel, so the finalize merge is shared.
//   copy warp      claims chunks, loads their metadata lane-parallel (required block, slot, bias,
//                  live tokens), and streams each K|V block (2 n_b d_head fp32) HBM -> shared
//                  memory with one 1-D bulk copy into a ring of NS stages; a chunk's query rows
//                  ride on its first block's barrier.
//   NW consumer    warps share every block.  QK for a group of 5..8 heads (TC): on the tensor
//   warps          cores in 3xTF32 (mma.m16n8k8: keys on M, heads on N; K tiles by ldmatrix from
//                  the swizzled stage; a = a_hi + a_lo, D += a_lo b_hi + a_hi b_lo + a_hi b_hi).
//                  Other group sizes: a key's dot products split over LPK lanes (DPL dims each,
//                  the queries in registers), reduced by a reduce-scatter butterfly (one lane per
//                  head ends with its sum).  Online softmax: one warp per head, accurate expf.
//                  PV in fp32 FMA: each warp owns NBK/NW keys and DH/32 dims per lane for every
//                  head; per-warp partials are rescaled per block and summed over the warps in a
//                  fixed tree at the chunk end (deterministic).
__device__ __forceinline__ int float_to_ordered(float f) {  // signed-int order == float order
  const int b = __float_as_int(f);
  return b ^ ((b >> 31) & 0x7fffffff);
}
__device__ __forceinline__ float ordered_to_float(int k) { return __int_as_float(k ^ ((k >> 31) & 0x7fffffff)); }
__device__ __forceinline__ unsigned f32_to_tf32(float x) {
  unsigned r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
// D = A(16x8 tf32, row) * B(8x8 tf32, col) + D, fp32 accumulate
__device__ __forceinline__ void mma_tf32(float (&c)[4], const unsigned (&a)[4], const unsigned (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

template <int NBK, int DH, int GP, int NW_ = 8>
struct F32W {
  static constexpr int NW = NW_;                    // consumer warps
  static constexpr int THREADS = (NW + 1) * 32;     // + the copy warp
  static constexpr int BPB = 2 * NBK * DH * 4;      // one K|V block
  static constexpr int PLANE = NBK * DH * 4;
  static constexpr int DPL = (GP >= 16 || NW >= 16) ? 4 : 8;  // QK dims per lane
  static constexpr int LPK = DH / DPL;              // lanes per key
  static constexpr int KPI = 32 / LPK;              // keys per warp iteration
  static constexpr int PCH = DPL / 4;               // 16-byte pieces per lane
  static constexpr int DPV = DH / 32;               // PV dims per lane
  static constexpr int QSLOT = GP * DH * 4;
  static constexpr int CB = 2;                      // partial buffers of the chunk-end tree
  // everything but the stages, the query slots and the unit table (cbase)
  static constexpr int SLD = NBK + 1;               // logit row stride (conflict-free writes)
  // QK on the tensor cores (3xTF32, mma.m16n8k8) for a group of 5..8 query heads: keys on M in
  // 16-row tiles, the heads on N = 8; with fewer tiles than warps the head dimension is split over
  // KS warps, each writing its own partial logits (summed in a fixed order by the softmax)
  static constexpr bool TC = GP == 8 && NW == 8;
  static constexpr int MT = NBK / 16;
  static constexpr int KS = TC ? (MT >= NW ? 1 : NW / MT) : 1;
  static constexpr int KSTEPS = DH / 8 / KS;       // k-steps of 8 dims per warp
  static constexpr int SPB = KS;                    // partial logit buffers
  static constexpr int FIXED = NBK * GP * 4 + SPB * (NBK * GP + GP) * 4 + CB * GP * DH * 4 + 3 * GP * 4 + 16 +
                               32 * 4 + 128;
  static constexpr int PER_STAGE = BPB + QSLOT + 16 + 20;
  // stages: as many as fit 227 KiB with 4 KiB left for the unit table, 2 to 4
  static constexpr int NS_FIT = (232448 - 4096 - FIXED) / PER_STAGE;
  static constexpr int NS = NS_FIT < 2 ? 2 : (NS_FIT > 4 ? 4 : NS_FIT);
  static size_t smem(int units) { return (size_t)FIXED + (size_t)NS * PER_STAGE + (size_t)(units + 1) * 4; }
  static_assert(GP <= LPK, "query heads per key group must not exceed its lanes");
  static_assert(NBK % NW == 0 || NBK < NW, "keys split over the warps");
};

struct F32Info {
  int bh, ci, count, flags;  // flags: 1 first block of its chunk, 2 last, 4 end of work
  float beta;
};

// Reduce-scatter butterfly of V values over the lanes of a key group.  Each lane holds its
// values in a lane-dependent order: slot j is query head j ^ m with m = dl / (LPK / GP) (the
// query rows are loaded permuted), so at every level the half a lane keeps is already its lower
// half: it sends the upper half and adds the partner's upper half, with no selects.  After the
// halving levels (offsets LPK/2 .. LPK/GP) slot 0 holds head m summed over the lanes that differ
// in those bits; the remaining levels are plain butterfly adds.
template <int V, int O>
struct RS {
  template <int N>
  static __device__ __forceinline__ void run(float (&v)[N]) {
    if constexpr (O >= 1) {
      if constexpr (V > 1) {
#pragma unroll
        for (int j = 0; j < V / 2; ++j) v[j] += __shfl_xor_sync(0xffffffffu, v[j + V / 2], O);
        RS<V / 2, O / 2>::run(v);
      } else {
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], O);
        RS<1, O / 2>::run(v);
      }
    }
  }
};

template <int NBK, int DH, int GP, int NW_>
__global__ void __launch_bounds__(F32W<NBK, DH, GP, NW_>::THREADS, 1)
    attend_f32w_kernel(Dev dv, int layer, int nl, const float* __restrict__ q, size_t q_layer_stride) {
  using T = F32W<NBK, DH, GP, NW_>;
  constexpr int NW = T::NW, LPK = T::LPK, KPI = T::KPI, DPL = T::DPL, DPV = T::DPV, NS = T::NS;
  extern __shared__ __align__(128) char smem_raw[];
  const int BHL = dv.B * dv.H;
  const int BH = nl * BHL;
  const int G = dv.G;
  char* p = smem_raw;
  char* stages = p;                                  p += (size_t)NS * T::BPB;
  char* qslots = p;                                  p += (size_t)NS * T::QSLOT;
  float* S = reinterpret_cast<float*>(p);            p += T::SPB * (NBK * GP + GP) * 4;  // [SPB][GP][NBK + 1] logits
  float* P = reinterpret_cast<float*>(p);            p += NBK * GP * 4;   // [NBK][GP] probabilities
  float* comb = reinterpret_cast<float*>(p);         p += T::CB * GP * DH * 4;
  float* run_m = reinterpret_cast<float*>(p);        p += GP * 4;
  float* run_l = reinterpret_cast<float*>(p);        p += GP * 4;
  float* scl = reinterpret_cast<float*>(p);          p += GP * 4;
  p = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
  uint64_t* full = reinterpret_cast<uint64_t*>(p);   p += NS * 8;
  uint64_t* empty = reinterpret_cast<uint64_t*>(p);  p += NS * 8;
  F32Info* info = reinterpret_cast<F32Info*>(p);     p += NS * sizeof(F32Info);
  int* tmp = reinterpret_cast<int*>(p);              p += 32 * 4;
  int* cbase = reinterpret_cast<int*>(p);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned long long t_start = dv.ktime ? globaltimer_ns() : 0ull;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    fence_mbar_init();
  }
  if (G < GP)  // query rows past the group stay zero (only G rows are copied in)
    for (int x = tid; x < NS * T::QSLOT / 16; x += blockDim.x) reinterpret_cast<int4*>(qslots)[x] = make_int4(0, 0, 0, 0);
  for (int g = tid; g < GP; g += blockDim.x) {
    run_m[g] = -INFINITY;
    run_l[g] = 0.0f;
  }
  chunk_scan(dv, layer, cbase, tmp, BH);  // also publishes the barrier inits (__syncthreads)
  const int total = cbase[BH];

  if (warp == NW) {
    // ------------------------------------------------------------ copy warp
    int seq = 0, cn = 0;
    int c = 0;
    if (lane == 0) c = atomicAdd(dv.cnt + kCntStride * layer + 1, 1);
    c = __shfl_sync(0xffffffffu, c, 0);
    while (c < total) {
      const int u = find_bh(cbase, BH, c);
      const int ci = c - cbase[u];
      const int lbh = layer * BHL + u;  // units of the launch's layers are contiguous in lbh
      const int rl = layer + u / BHL, bh = u % BHL;
      const int n = __ldcg(dv.n_req + lbh);
      const int t = __ldcg(dv.t + lbh);
      const int i0 = ci * dv.chunk, nb = min(dv.chunk, n - i0);
      // the chunk's blocks, lane-parallel: block, slot, bias, live tokens
      int blk = 0, slot = 0, cnt = 0;
      float beta = 0.0f;
      if (lane < nb) {
        blk = __ldcg(dv.req + (size_t)lbh * dv.C + i0 + lane);
        slot = __ldcg(dv.req_slot + (size_t)lbh * dv.C + i0 + lane);
        cnt = min(NBK, t - blk * NBK);
        beta = block_beta(dv, lbh, blk, t);
      }
      // the next chunk's claim is in flight while this one streams
      int c_next = 0;
      if (lane == 0) c_next = atomicAdd(dv.cnt + kCntStride * layer + 1, 1);
      const int b = bh / dv.H, h = bh % dv.H;
      const float* qrow = q + (size_t)(rl - layer) * q_layer_stride + ((size_t)b * dv.Hq + h * G) * DH;
      for (int i = 0; i < nb; ++i, ++seq) {
        const int st = seq % NS;
        const int si = __shfl_sync(0xffffffffu, slot, i);
        const int ki = __shfl_sync(0xffffffffu, cnt, i);
        const float be = __shfl_sync(0xffffffffu, beta, i);
        if (lane == 0) {
          if (seq >= NS) mbar_wait(&empty[st], ((seq / NS) - 1) & 1);
          info[st] = F32Info{u, ci, ki, (i == 0 ? 1 : 0) | (i == nb - 1 ? 2 : 0), be};
          fence_proxy_async();
          const unsigned qbytes = i == 0 ? (unsigned)(G * DH * 4) : 0u;
          mbar_expect_tx(&full[st], T::BPB + qbytes);
          bulk_g2s(stages + (size_t)st * T::BPB, dv.pool + ((size_t)lbh * dv.C + si) * (size_t)T::BPB, T::BPB, &full[st]);
          if (qbytes) bulk_g2s(qslots + (size_t)(cn % NS) * T::QSLOT, qrow, qbytes, &full[st]);
        }
      }
      ++cn;
      c = __shfl_sync(0xffffffffu, c_next, 0);
    }
    if (lane == 0) {  // end of work
      const int st = seq % NS;
      if (seq >= NS) mbar_wait(&empty[st], ((seq / NS) - 1) & 1);
      info[st] = F32Info{-1, 0, 0, 4, 0.0f};
      mbar_arrive_plain(&full[st]);
    }
  } else {
    // ------------------------------------------------------------ consumer warps
    const int dl = lane % LPK, kq = lane / LPK;
    const int qperm = dl / (LPK / GP);  // this lane's register slot j holds query head j ^ qperm
    float qr[T::TC ? 1 : GP][T::TC ? 1 : DPL];
    unsigned qhi[T::TC ? T::KSTEPS : 1][2], qlo[T::TC ? T::KSTEPS : 1][2];  // B fragments (TC)
    const int gid = lane >> 2, tig = lane & 3;
    const int tc_mt = warp % T::MT, tc_kp = warp / T::MT;  // TC: key tile, head-dimension part
    float o[GP][DPV];
#pragma unroll
    for (int g = 0; g < GP; ++g)
#pragma unroll
      for (int x = 0; x < DPV; ++x) o[g][x] = 0.0f;
    constexpr int NHW = (GP + NW - 1) / NW;  // query heads per softmax warp
    float mreg[NHW], lpart[NHW];
#pragma unroll
    for (int j = 0; j < NHW; ++j) {
      mreg[j] = -INFINITY;
      lpart[j] = 0.0f;
    }
    int seq = 0, cn = 0;
    for (;; ++seq) {
      const int st = seq % NS;
      mbar_wait(&full[st], (seq / NS) & 1);
      const F32Info it = info[st];
      if (it.flags & 4) break;
      const char* kb = stages + (size_t)st * T::BPB;
      const char* vb = kb + T::PLANE;
      if (it.flags & 1) {  // chunk start: the group's query slice into registers
        const float* qs = reinterpret_cast<const float*>(qslots + (size_t)(cn % NS) * T::QSLOT);
        if constexpr (T::TC) {
#pragma unroll
          for (int k = 0; k < T::KSTEPS; ++k)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const float x = qs[gid * DH + 8 * (tc_kp * T::KSTEPS + k) + tig + 4 * e];
              qhi[k][e] = f32_to_tf32(x);
              qlo[k][e] = f32_to_tf32(x - __uint_as_float(qhi[k][e]));
            }
        } else {
#pragma unroll
          for (int g = 0; g < GP; ++g)
#pragma unroll
            for (int j = 0; j < DPL / 4; ++j) {
              const float4 v4 = *reinterpret_cast<const float4*>(qs + (g ^ qperm) * DH + 4 * (dl + j * LPK));
              qr[g][4 * j] = v4.x;
              qr[g][4 * j + 1] = v4.y;
              qr[g][4 * j + 2] = v4.z;
              qr[g][4 * j + 3] = v4.w;
            }
        }
      }
      const int count = it.count;
      if constexpr (T::TC) {
        // ---- QK on the tensor cores: this warp's 16-key tile x the group's 8 heads over its
        //      k-steps; a = a_hi + a_lo in tf32 for K and q, D += a_lo b_hi + a_hi b_lo + a_hi b_hi
        // four independent accumulators (k-step parity x {cross terms, hi.hi}) keep the MMA
        // dependency chains short; summed in a fixed order after the k loop
        float c4[4][4] = {};
        const int mi = lane >> 3, r = lane & 7;
        const int key_a = tc_mt * 16 + r + (mi & 1) * 8;
        const unsigned rowb = smem_u32(kb) + key_a * DH * 4;
#pragma unroll
        for (int k = 0; k < T::KSTEPS; ++k) {
          const int chunk = 2 * (tc_kp * T::KSTEPS + k) + (mi >> 1);
          unsigned a[4];
          ldsm_x4(rowb + ((chunk ^ (key_a & 7)) << 4), a[0], a[1], a[2], a[3]);
          // split in integer ops: hi = x rounded to the tf32 grid (round half away from zero on
          // the magnitude), lo = x - hi exactly; the tensor core reads lo's top 19 bits
          unsigned ahi[4], alo[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            ahi[e] = (a[e] + 0x1000u) & 0xffffe000u;
            alo[e] = __float_as_uint(__uint_as_float(a[e]) - __uint_as_float(ahi[e]));
          }
          mma_tf32(c4[2 * (k & 1)], alo, qhi[k]);
          mma_tf32(c4[2 * (k & 1)], ahi, qlo[k]);
          mma_tf32(c4[2 * (k & 1) + 1], ahi, qhi[k]);
        }
        float c[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) c[e] = (c4[0][e] + c4[2][e]) + (c4[1][e] + c4[3][e]);
        float* Sp = S + (size_t)tc_kp * (NBK * GP + GP);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int key = tc_mt * 16 + gid + (e >> 1) * 8, g = 2 * tig + (e & 1);
          Sp[g * T::SLD + key] = c[e];
        }
      } else {
      // ---- QK: logits + bias into S[g][key] (keys past the live tokens: -inf); every K load of
      //      the warp's keys is issued before the first FMA
      constexpr int NIT = (NBK + NW * KPI - 1) / (NW * KPI);
      constexpr int PFI = GP >= 16 ? (NIT < 2 ? NIT : 2) : NIT;  // iterations whose K loads go out together
#pragma unroll
      for (int i0 = 0; i0 < NIT; i0 += PFI) {
        if ((i0 * NW + warp) * KPI >= NBK) break;  // warp-uniform
        float4 k4[PFI][DPL / 4];
#pragma unroll
        for (int ii = 0; ii < PFI; ++ii) {
          const int key = ((i0 + ii) * NW + warp) * KPI + kq;
#pragma unroll
          for (int j = 0; j < DPL / 4; ++j) {
            const int chunk = dl + j * LPK;
            k4[ii][j] = key < count ? *reinterpret_cast<const float4*>(kb + key * DH * 4 + ((chunk ^ (key & 7)) << 4))
                                    : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
          }
        }
#pragma unroll
        for (int ii = 0; ii < PFI; ++ii) {
          const int i = i0 + ii;
          const int key = (i * NW + warp) * KPI + kq;
          if (i >= NIT || (i * NW + warp) * KPI >= NBK) break;  // warp-uniform
          float v[GP];
#pragma unroll
          for (int g = 0; g < GP; ++g) v[g] = 0.0f;
#pragma unroll
          for (int j = 0; j < DPL / 4; ++j)
#pragma unroll
            for (int g = 0; g < GP; ++g) {
              v[g] = fmaf(qr[g][4 * j], k4[ii][j].x, v[g]);
              v[g] = fmaf(qr[g][4 * j + 1], k4[ii][j].y, v[g]);
              v[g] = fmaf(qr[g][4 * j + 2], k4[ii][j].z, v[g]);
              v[g] = fmaf(qr[g][4 * j + 3], k4[ii][j].w, v[g]);
            }
          RS<GP, LPK / 2>::run(v);
          if (dl % (LPK / GP) == 0 && key < NBK && qperm < G)
            S[qperm * T::SLD + key] = v[0];
        }
      }
      }
      named_sync(kBarConsumers, NW * 32);
      // ---- online softmax, one warp per query head: the running max in a register, the running
      //      sum as per-lane partials (reduced across the lanes once, at the chunk end)
#pragma unroll
      for (int j = 0; j < NHW; ++j) {
        const int g = warp + NW * j;
        if (g >= G) break;
        float sv[(NBK + 31) / 32];
        float mx = -INFINITY;
#pragma unroll
        for (int r = 0; r < (NBK + 31) / 32; ++r) {
          const int key = lane + 32 * r;
          float x = 0.0f;
#pragma unroll
          for (int pp = 0; pp < T::SPB; ++pp) x += key < NBK ? S[pp * (NBK * GP + GP) + g * T::SLD + key] : 0.0f;
          sv[r] = key < count ? x + it.beta : -INFINITY;
          mx = fmaxf(mx, sv[r]);
        }
        // warp max in one REDUX on the order-preserving integer image of the float
        mx = ordered_to_float(__reduce_max_sync(0xffffffffu, float_to_ordered(mx)));
        const float m_old = mreg[j];
        const float mn = fmaxf(m_old, mx);
        const float sc = expf(m_old - mn);
        float sum = 0.0f;
#pragma unroll
        for (int r = 0; r < (NBK + 31) / 32; ++r) {
          const int key = lane + 32 * r;
          const float pr = expf(sv[r] - mn);
          if (key < NBK) P[key * GP + g] = pr;
          sum += key < NBK ? pr : 0.0f;
        }
        lpart[j] = lpart[j] * sc + sum;
        mreg[j] = mn;
        if (lane == 0) scl[g] = sc;
      }
      named_sync(kBarConsumers, NW * 32);
      // ---- PV over this warp's keys, after rescaling its partial to the new running max
#pragma unroll
      for (int g = 0; g < GP; ++g) {
        const float sc = g < G ? scl[g] : 0.0f;
#pragma unroll
        for (int x = 0; x < DPV; ++x) o[g][x] *= sc;
      }
      constexpr int KPW = (NBK + NW - 1) / NW;  // keys per warp: warp, warp + NW, ...
      // with NW a multiple of 8 every key of this warp has the same swizzle phase (key & 7)
      const char* vrow = vb + warp * DH * 4;
      const float* prow = P + warp * GP;
#pragma unroll
      for (int j = 0; j < KPW; ++j) {
        const int key = warp + NW * j;
        if (key >= count) break;  // warp-uniform
        float vv[DPV];
        if constexpr (DPV == 4) {
          const int sw = (NW % 8 == 0) ? (warp & 7) : (key & 7);
          const float4 v4 = *reinterpret_cast<const float4*>(vrow + j * NW * DH * 4 + ((lane ^ sw) << 4));
          vv[0] = v4.x; vv[1] = v4.y; vv[2] = v4.z; vv[3] = v4.w;
        } else {
          const float2 v2 = *reinterpret_cast<const float2*>(vb + swz_off(key, DPV * lane, DH, 4));
          vv[0] = v2.x; vv[1] = v2.y;
        }
        const float* pk = prow + j * NW * GP;
#pragma unroll
        for (int g4 = 0; g4 < GP; g4 += 4) {
          const float4 p4 = *reinterpret_cast<const float4*>(pk + g4);
          const float pp[4] = {p4.x, p4.y, p4.z, p4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e)
#pragma unroll
            for (int x = 0; x < DPV; ++x) o[g4 + e][x] = fmaf(pp[e], vv[x], o[g4 + e][x]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      if (it.flags & 2) {
        // ---- chunk end: each softmax warp publishes its heads' (m, l), l summed over the lanes
        //      in a fixed butterfly; then the warps' partial O are summed in a fixed tree (warp w
        //      += warp w + half, CB pairs at a time through the partial buffers), and warp 0 writes
        //      the record (the tree's barriers order the (m, l) stores before its reads)
#pragma unroll
        for (int j = 0; j < NHW; ++j) {
          const int g = warp + NW * j;
          if (g >= G) break;
          float l = lpart[j];
#pragma unroll
          for (int off = 16; off; off >>= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
          if (lane == 0) {
            run_m[g] = mreg[j];
            run_l[g] = l;
          }
          mreg[j] = -INFINITY;
          lpart[j] = 0.0f;
        }
        for (int half = NW / 2; half >= 1; half >>= 1) {
          for (int p0 = 0; p0 < half; p0 += T::CB) {
            const int p1 = min(p0 + T::CB, half);
            if (warp >= half + p0 && warp < half + p1) {
              float* cw = comb + (size_t)(warp - half - p0) * GP * DH;
#pragma unroll
              for (int g = 0; g < GP; ++g) {
                if constexpr (DPV == 4)
                  *reinterpret_cast<float4*>(cw + g * DH + 4 * lane) = make_float4(o[g][0], o[g][1], o[g][2], o[g][3]);
                else
                  *reinterpret_cast<float2*>(cw + g * DH + 2 * lane) = make_float2(o[g][0], o[g][1]);
              }
            }
            named_sync(kBarConsumers, NW * 32);
            if (warp >= p0 && warp < p1) {
              const float* cw = comb + (size_t)(warp - p0) * GP * DH;
#pragma unroll
              for (int g = 0; g < GP; ++g) {
                if constexpr (DPV == 4) {
                  const float4 c4 = *reinterpret_cast<const float4*>(cw + g * DH + 4 * lane);
                  o[g][0] += c4.x; o[g][1] += c4.y; o[g][2] += c4.z; o[g][3] += c4.w;
                } else {
                  const float2 c2 = *reinterpret_cast<const float2*>(cw + g * DH + 2 * lane);
                  o[g][0] += c2.x; o[g][1] += c2.y;
                }
              }
            }
            named_sync(kBarConsumers, NW * 32);
          }
        }
        if (warp == 0) {
          const int u = it.bh, rl = layer + u / BHL;
          const size_t pbase = (size_t)(u % BHL) * dv.max_chunks + it.ci;
          float* po = part_o_of(dv, rl);
#pragma unroll
          for (int g = 0; g < GP; ++g) {
            if (g >= G) break;
            if constexpr (DPV == 4)
              *reinterpret_cast<float4*>(po + (pbase * G + g) * DH + 4 * lane) = make_float4(o[g][0], o[g][1], o[g][2], o[g][3]);
            else
              *reinterpret_cast<float2*>(po + (pbase * G + g) * DH + 2 * lane) = make_float2(o[g][0], o[g][1]);
          }
          if (lane < G) part_ml_of(dv, rl)[pbase * G + lane] = make_float2(run_m[lane], run_l[lane]);
        }
#pragma unroll
        for (int g = 0; g < GP; ++g)
#pragma unroll
          for (int x = 0; x < DPV; ++x) o[g][x] = 0.0f;
        ++cn;
      }
    }
  }
  if (dv.ktime) {  // diagnostics: device-clock span of the launch (first CTA start .. last CTA end)
    __syncthreads();
    if (tid == 0) {
      atomicMin(dv.ktime + 2 * layer, t_start);
      atomicMax(dv.ktime + 2 * layer + 1, globaltimer_ns());
    }
  }
}

// ---------------------------------------------------------------- finalize (merge + append)
// One CTA per (b, h): log-sum-exp merge of the chunk records in chunk order, then the append.
// Runs after the attention kernel of the layer, so every chunk record is complete and no
// thread can still be reading the tail block.
template <typename T>
__global__ void __launch_bounds__(kFinThreads)
    finalize_kernel(Dev dv, int layer0, const T* __restrict__ kn0, const T* __restrict__ vn0, float* __restrict__ out0) {
  // grid (B*H, layers): layer = layer0 + blockIdx.y, its k/v rows and outputs one layer stride on
  extern __shared__ __align__(16) char fin_smem[];
  double* zsm = reinterpret_cast<double*>(fin_smem);           // [n_ev]
  float* wsm = reinterpret_cast<float*>(zsm + dv.n_ev);         // [kFinThreads] f64 reduction scratch
  const int bh = blockIdx.x, layer = layer0 + blockIdx.y;
  const size_t kst = (size_t)dv.B * dv.H * dv.D, ost = (size_t)dv.B * dv.Hq * dv.D;
  finalize_bh<T>(dv, layer, bh, kn0 + blockIdx.y * kst, vn0 + blockIdx.y * kst, out0 + blockIdx.y * ost, wsm, zsm);
}

// layers [layer, layer + nl): kn/vn/out point at layer `layer`'s rows
cudaError_t launch_finalize(const Dev& dv, int layer, const void* kn, const void* vn, float* out, cudaStream_t st,
                            int nl) {
  const size_t smem = (size_t)dv.n_ev * 8 + (size_t)kFinThreads * 8;
  const dim3 grid(dv.B * dv.H, nl);
  if (dv.dtype == 0) {
    auto k = finalize_kernel<__nv_bfloat16>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    max_shared_carveout(k);
    k<<<grid, kFinThreads, smem, st>>>(dv, layer, static_cast<const __nv_bfloat16*>(kn),
                                        static_cast<const __nv_bfloat16*>(vn), out);
  } else {
    auto k = finalize_kernel<float>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    max_shared_carveout(k);
    k<<<grid, kFinThreads, smem, st>>>(dv, layer, static_cast<const float*>(kn), static_cast<const float*>(vn), out);
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------- launchers
template <int NBK, int DH, int NQT>
static cudaError_t launch_bf16(const Dev& dv, int layer, int nl, const void* q, cudaStream_t st, int num_sms) {
  using T = BF<NBK, DH, NQT>;
  const int BH = nl * dv.B * dv.H;
  const size_t smem = bf_smem_fixed<NBK, DH, NQT>() + (size_t)(BH + 1) * 4 + 64;
  auto k = attend_bf16_kernel<NBK, DH, NQT>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  max_shared_carveout(k);
  k<<<num_sms, T::THREADS, smem, st>>>(dv, layer, nl, static_cast<const __nv_bfloat16*>(q),
                                       (size_t)dv.B * dv.Hq * DH);
  return cudaGetLastError();
}

template <int NBK, int DH>
static cudaError_t launch_f32(const Dev& dv, int layer, const void* q, const void* kn, const void* vn, float* out,
                              cudaStream_t st, int num_sms) {
  constexpr int NS = 2;
  constexpr int BPB = 2 * NBK * DH * 4;
  const int BH = dv.B * dv.H;
  const size_t smem = (size_t)NS * BPB + NS * 8 + 16 * DH * 4 + 16 * NBK * 4 + (NS + 2) * 4 + 32 * 4 +
                      (BH + 1) * 4 + 64;
  auto k = attend_f32_kernel<NBK, DH, NS>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k<<<num_sms, 32, smem, st>>>(dv, layer, static_cast<const float*>(q), static_cast<const float*>(kn),
                               static_cast<const float*>(vn), out);
  return cudaGetLastError();
}

template <int NBK, int DH, int GP, int NW = 8>
static cudaError_t launch_f32w(const Dev& dv, int layer, int nl, const void* q, cudaStream_t st, int num_sms) {
  using T = F32W<NBK, DH, GP, NW>;
  const size_t smem = T::smem(nl * dv.B * dv.H);
  if (smem > 232448) return cudaErrorInvalidConfiguration;  // unit table too large for one launch
  auto k = attend_f32w_kernel<NBK, DH, GP, NW>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  max_shared_carveout(k);
  k<<<num_sms, T::THREADS, smem, st>>>(dv, layer, nl, static_cast<const float*>(q), (size_t)dv.B * dv.Hq * DH);
  return cudaGetLastError();
}

static bool f32_single_warp() {  // the round-1 one-warp fp32 kernel, one layer per launch (A/B)
  static const bool v = getenv("NOSA_F32_WARP") != nullptr;
  return v;
}

template <int NBK, int DH>
static cudaError_t dispatch_f32(const Dev& dv, int layer, int nl, const void* q, const void* kn, const void* vn,
                                float* out, cudaStream_t st, int num_sms) {
  if (f32_single_warp()) {
    if (nl != 1) return cudaErrorInvalidValue;
    return launch_f32<NBK, DH>(dv, layer, q, kn, vn, out, st, 2 * num_sms);
  }
  static const bool w16 = getenv("NOSA_F32_WARPS16") != nullptr;  // A/B: 16 consumer warps, 4 dims per lane
  if (w16 && NBK == 64 && DH == 128 && dv.G > 4 && dv.G <= 8) return launch_f32w<NBK, DH, 8, 16>(dv, layer, nl, q, st, num_sms);
  if (dv.G <= 4) return launch_f32w<NBK, DH, 4>(dv, layer, nl, q, st, num_sms);
  if (dv.G <= 8) return launch_f32w<NBK, DH, 8>(dv, layer, nl, q, st, num_sms);
  return launch_f32w<NBK, DH, 16>(dv, layer, nl, q, st, num_sms);
}

bool attend_f32_per_layer() { return f32_single_warp(); }

bool attend_supported(int n_b, int d_head, int dtype) {
  const bool nb_ok = n_b == 16 || n_b == 32 || n_b == 64 || n_b == 128;
  const bool d_ok = d_head == 64 || d_head == 128;
  if (dtype == 1 && n_b == 128 && d_head == 128) return false;  // 128 KiB fp32 blocks: no double buffer
  return nb_ok && d_ok;
}

template <int NBK, int DH>
static cudaError_t dispatch_bf16(const Dev& dv, int layer, int nl, const void* q, cudaStream_t st, int num_sms) {
  return dv.G <= 8 ? launch_bf16<NBK, DH, 1>(dv, layer, nl, q, st, num_sms)
                   : launch_bf16<NBK, DH, 2>(dv, layer, nl, q, st, num_sms);
}

// layers [layer, layer + nl) in one launch (bf16 and the fp32 warp-group kernel; the one-warp fp32
// kernel of NOSA_F32_WARP=1 runs one layer at a time)
cudaError_t launch_attend(const Dev& dv, int layer, int nl, const void* q, const void* kn, const void* vn, float* out,
                          cudaStream_t st, int num_sms) {
#define NOSA_DISPATCH(NBK, DH)                                                                  \
  if (dv.n_b == NBK && dv.D == DH) {                                                            \
    return dv.dtype == 0 ? dispatch_bf16<NBK, DH>(dv, layer, nl, q, st, num_sms)                \
                         : dispatch_f32<NBK, DH>(dv, layer, nl, q, kn, vn, out, st, num_sms);   \
  }
  NOSA_DISPATCH(64, 128)
  NOSA_DISPATCH(64, 64)
  NOSA_DISPATCH(32, 128)
  NOSA_DISPATCH(32, 64)
  NOSA_DISPATCH(16, 128)
  NOSA_DISPATCH(16, 64)
  NOSA_DISPATCH(128, 64)
  if (dv.n_b == 128 && dv.D == 128 && dv.dtype == 0) return dispatch_bf16<128, 128>(dv, layer, nl, q, st, num_sms);
#undef NOSA_DISPATCH
  return cudaErrorInvalidValue;
}

}  // namespace nosa
