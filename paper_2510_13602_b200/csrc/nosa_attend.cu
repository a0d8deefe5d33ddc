// nosa_attend.cu — K4 block-sparse biased decode attention + K5 append.
//
// Restates, per (sequence, kv head), the attention half of DecodeEngine.step
// (decode.py:178-185): for each query head of the GQA group, softmax over the attended
// tokens of  q.k_j + beta_j  (unscaled logits, attention.py:180) with beta_j the block-mean
// eviction score of token j's block (decode.py:180-181, 192-194; bias_logit_offsets
// attention.py:149-164), then w.V.  Masked tokens (outside Gamma(t)) contribute exactly zero,
// so only the required blocks are read; the partial tail block is clipped at t
// (selection.py:104-107).  After attention the new token is appended (decode.py:187-189) with
// its ed-dma importance score (importance_scores, attention.py:121-146).
//
// Work decomposition: each (b, h) required list is cut into chunks of kChunk blocks (fixed
// split, so results do not depend on grid size or batch composition).  A persistent grid of
// warps claims chunks from a per-layer counter; every warp streams its blocks through a
// private ring of shared-memory stages filled by 1-D TMA bulk copies (cp.async.bulk, one
// 32 KiB K|V block per copy, mbarrier completion).  bf16: QK^T and PV on tensor cores
// (mma.m16n8k16, queries on M padded to 16, keys/dims on N), online softmax in registers.
// The last warp to finish a (b, h) merges the chunk partials in chunk order (log-sum-exp) and
// performs the append, so no other warp can still be reading the tail block.
#include "nosa_device.cuh"

namespace nosa {

constexpr float kLog2e = 1.4426950408889634f;

struct AttnShared {
  int* cbase;   // [BH + 1] exclusive prefix of chunk counts
  int* ring;    // [NW][RING] claimed chunk ids per warp
};

// per-item geometry
struct Item {
  int bh, lbh, i;
};

__device__ __forceinline__ int find_bh(const int* cbase, int BH, int c) {
  int lo = 0, hi = BH;  // largest bh with cbase[bh] <= c
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (cbase[mid] <= c) lo = mid; else hi = mid;
  }
  return lo;
}

// block-level exclusive scan of ceil(n_req/kChunk) over BH entries into cbase
__device__ void chunk_scan(const Dev& dv, int layer, int* cbase, int* tmp) {
  const int BH = dv.B * dv.H;
  const int nt = blockDim.x;
  const int per = (BH + nt - 1) / nt;
  const int lo = threadIdx.x * per, hi = min(BH, lo + per);
  int s = 0;
  for (int i = lo; i < hi; ++i) s += (dv.n_req[layer * BH + i] + kChunk - 1) / kChunk;
  tmp[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int i = 0; i < nt; ++i) {
      const int v = tmp[i];
      tmp[i] = acc;
      acc += v;
    }
    cbase[BH] = acc;
  }
  __syncthreads();
  int acc = tmp[threadIdx.x];
  for (int i = lo; i < hi; ++i) {
    cbase[i] = acc;
    acc += (dv.n_req[layer * BH + i] + kChunk - 1) / kChunk;
  }
  __syncthreads();
}

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

// ---------------------------------------------------------------- merge + append (one warp)
template <typename T>
__device__ void merge_and_append(const Dev& dv, int layer, int bh, int nc, const T* __restrict__ kn,
                                 const T* __restrict__ vn, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int b = bh / dv.H, h = bh % dv.H;
  const int lbh = (layer * dv.B + b) * dv.H + h;
  const int D = dv.D, G = dv.G;
  __threadfence();
  // ---- merge chunk partials in chunk order (deterministic)
  for (int g = 0; g < G; ++g) {
    float M = -INFINITY;
    for (int c = 0; c < nc; ++c) M = fmaxf(M, __ldcg(&dv.part_ml[((size_t)bh * dv.max_chunks + c) * G + g]).x);
    float Lsum = 0.0f;
    for (int c = 0; c < nc; ++c) {
      const float2 ml = __ldcg(&dv.part_ml[((size_t)bh * dv.max_chunks + c) * G + g]);
      Lsum += ml.y * expf(ml.x - M);
    }
    const float inv = 1.0f / Lsum;
    for (int d = lane; d < D; d += 32) {
      float acc = 0.0f;
      for (int c = 0; c < nc; ++c) {
        const float w = expf(__ldcg(&dv.part_ml[((size_t)bh * dv.max_chunks + c) * G + g]).x - M);
        acc += w * __ldcg(&dv.part_o[(((size_t)bh * dv.max_chunks + c) * G + g) * D + d]);
      }
      out[((size_t)b * dv.Hq + h * G + g) * D + d] = acc * inv;
    }
  }
  // ---- append the new token (decode.py:187-189, HeadState.append decode.py:65-71)
  const int t = dv.t[lbh];
  const int n_b = dv.n_b;
  const int blk = t / n_b, r = t - blk * n_b;
  const T* kr = kn + ((size_t)b * dv.H + h) * D;
  const T* vr = vn + ((size_t)b * dv.H + h) * D;
  const int elem = dv.elem;
  const int plane = n_b * D * elem;
  const int slot = dv.slot_of[(size_t)lbh * dv.NB + blk];
  char* hblk = dv.host + ((size_t)lbh * dv.NB + blk) * dv.bpb;
  char* dblk = slot >= 0 ? dv.pool + ((size_t)lbh * dv.C + slot) * dv.bpb : nullptr;
  const int chunks_per_row = D * elem / 16;
  for (int c = lane; c < 2 * chunks_per_row; c += 32) {
    const int which = c / chunks_per_row;  // 0 = K, 1 = V
    const int ch = c - which * chunks_per_row;
    const int4 val = reinterpret_cast<const int4*>(which ? (const void*)vr : (const void*)kr)[ch];
    const int off = which * plane + r * D * elem + ((ch ^ (r & 7)) << 4);
    *reinterpret_cast<int4*>(hblk + off) = val;
    if (dblk) *reinterpret_cast<int4*>(dblk + off) = val;
  }
  if (r == 0) {  // a new block: the slow copy of its unwritten rows must read as zero
    const int4 z = make_int4(0, 0, 0, 0);
    const int row_chunks = D * elem / 16;
    const int total = 2 * (n_b - 1) * row_chunks;
    for (int c = lane; c < total; c += 32) {
      const int which = c / ((n_b - 1) * row_chunks);
      const int rem = c - which * (n_b - 1) * row_chunks;
      const int row = 1 + rem / row_chunks;
      const int ch = rem % row_chunks;
      *reinterpret_cast<int4*>(hblk + which * plane + row * D * elem + (ch << 4)) = z;
    }
  }
  // importance score of the new token and the tail-block running means
  const double s = token_score_warp<T>(vr, dv.w1, dv.w2, D, dv.n_ev, dv.variant);
  double* tks = dv.tail_ksum + (size_t)lbh * D;
  for (int d = lane; d < D; d += 32) {
    const double kv = to_f64(kr[d]);
    const double acc = (r == 0) ? kv : tks[d] + kv;
    if (r == n_b - 1) {
      dv.kc[((size_t)lbh * dv.NB + blk) * D + d] = acc / (double)n_b;
      tks[d] = 0.0;
    } else {
      tks[d] = acc;
    }
  }
  if (lane == 0) {
    const double acc = (r == 0) ? s : dv.tail_se[lbh] + s;
    if (r == n_b - 1) {
      dv.se[(size_t)lbh * dv.NB + blk] = acc / (double)n_b;
      dv.tail_se[lbh] = 0.0;
    } else {
      dv.tail_se[lbh] = acc;
    }
    dv.t[lbh] = t + 1;
  }
  __threadfence_system();
}

// ---------------------------------------------------------------- bf16 tensor-core kernel
template <int NBK, int DH, int NW, int NS>
__global__ void __launch_bounds__(NW * 32)
    attend_bf16_kernel(Dev dv, int layer, const __nv_bfloat16* __restrict__ q,
                       const __nv_bfloat16* __restrict__ kn, const __nv_bfloat16* __restrict__ vn,
                       float* __restrict__ out) {
  constexpr int BPB = 2 * NBK * DH * 2;
  constexpr int PLANE = NBK * DH * 2;
  constexpr int RING = NS + 2;
  constexpr int NT = NBK / 8;   // key n-tiles
  constexpr int KS = DH / 16;   // k-steps over head dims
  constexpr int ON = DH / 8;    // output n-tiles
  extern __shared__ __align__(128) char smem_raw[];
  const int BH = dv.B * dv.H;
  char* stages = smem_raw;                                          // [NW][NS][BPB]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + (size_t)NW * NS * BPB);  // [NW][NS]
  int* cbase = reinterpret_cast<int*>(bars + NW * NS);              // [BH+1]
  int* ring = cbase + BH + 1;                                       // [NW][RING]
  int* tmp = ring + NW * RING;                                      // [blockDim]

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  if (lane == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bars[warp * NS + s], 1);
    fence_mbar_init();
  }
  chunk_scan(dv, layer, cbase, tmp);
  const int total = cbase[BH];
  __syncwarp();

  char* my_stages = stages + (size_t)warp * NS * BPB;
  uint64_t* my_bars = bars + warp * NS;
  int* my_ring = ring + warp * RING;

  // loader state (warp-uniform)
  int ld_seq = 0, ld_chunk_n = 0;       // items issued, chunks claimed
  int ld_bh = 0, ld_i = 0, ld_end = 0;  // current loader chunk
  bool ld_done = false;
  auto advance_loader = [&]() {
    if (ld_done) return;
    if (ld_i >= ld_end) {
      int c = 0;
      if (lane == 0) c = atomicAdd(dv.cnt + 2 * layer + 1, 1);
      c = __shfl_sync(0xffffffffu, c, 0);
      if (c >= total) { ld_done = true; return; }
      ld_bh = find_bh(cbase, BH, c);
      const int ci = c - cbase[ld_bh];
      const int nreq = dv.n_req[layer * BH + ld_bh];
      ld_i = ci * kChunk;
      ld_end = min(ld_i + kChunk, nreq);
      if (lane == 0) my_ring[ld_chunk_n % RING] = c;
      ++ld_chunk_n;
    }
    const int lbh = layer * BH + ld_bh;
    const int slot = dv.req_slot[(size_t)lbh * dv.C + ld_i];
    const int st = ld_seq % NS;
    if (lane == 0) {
      fence_proxy_async();
      mbar_expect_tx(&my_bars[st], BPB);
      bulk_g2s(my_stages + (size_t)st * BPB, dv.pool + ((size_t)lbh * dv.C + slot) * (size_t)BPB, BPB,
               &my_bars[st]);
    }
    ++ld_i;
    ++ld_seq;
  };

  for (int s = 0; s < NS; ++s) advance_loader();
  __syncwarp();

  int cp_seq = 0, cp_chunk_n = 0;
  int cp_bh = 0, cp_i = 0, cp_end = 0, cp_c = 0, cp_ci = 0;
  int cp_t = 0;
  unsigned qa[KS][4];
  float o[ON][4];
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.0f, l1 = 0.0f;
  const bool v0 = g < dv.G, v1 = (g + 8) < dv.G;

  while (cp_seq < ld_seq) {
    if (cp_i >= cp_end) {  // start of a new chunk
      __syncwarp();
      cp_c = my_ring[cp_chunk_n % RING];
      ++cp_chunk_n;
      cp_bh = find_bh(cbase, BH, cp_c);
      cp_ci = cp_c - cbase[cp_bh];
      const int nreq = dv.n_req[layer * BH + cp_bh];
      cp_i = cp_ci * kChunk;
      cp_end = min(cp_i + kChunk, nreq);
      const int b = cp_bh / dv.H, h = cp_bh % dv.H;
      cp_t = dv.t[layer * BH + cp_bh];
      const __nv_bfloat16* qb = q + ((size_t)b * dv.Hq + h * dv.G) * DH;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int c0 = ks * 16 + 2 * tq;
        qa[ks][0] = v0 ? *reinterpret_cast<const unsigned*>(qb + (size_t)g * DH + c0) : 0u;
        qa[ks][1] = v1 ? *reinterpret_cast<const unsigned*>(qb + (size_t)(g + 8) * DH + c0) : 0u;
        qa[ks][2] = v0 ? *reinterpret_cast<const unsigned*>(qb + (size_t)g * DH + c0 + 8) : 0u;
        qa[ks][3] = v1 ? *reinterpret_cast<const unsigned*>(qb + (size_t)(g + 8) * DH + c0 + 8) : 0u;
      }
#pragma unroll
      for (int n = 0; n < ON; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.0f;
      m0 = m1 = -INFINITY;
      l0 = l1 = 0.0f;
    }
    const int lbh = layer * BH + cp_bh;
    const int blk = dv.req[(size_t)lbh * dv.C + cp_i];
    const int count = min(NBK, cp_t - blk * NBK);
    const float beta = block_beta(dv, lbh, blk, cp_t);
    const int st = cp_seq % NS;
    mbar_wait(&my_bars[st], (cp_seq / NS) & 1);
    const unsigned kbase = smem_u32(my_stages + (size_t)st * BPB);
    const unsigned vbase = kbase + PLANE;

    // ---- S = Q K^T  (rows: query heads, cols: keys)
    float s[NT][4];
#pragma unroll
    for (int j = 0; j < NT; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.0f;
#pragma unroll
    for (int p = 0; p < KS / 2; ++p) {
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const int row = j * 8 + (lane & 7);
        const int chunk = p * 4 + (lane >> 3);
        unsigned b0, b1, b2, b3;
        ldsm_x4(kbase + row * (DH * 2) + ((chunk ^ (row & 7)) << 4), b0, b1, b2, b3);
        mma_bf16(s[j], qa[2 * p][0], qa[2 * p][1], qa[2 * p][2], qa[2 * p][3], b0, b1);
        mma_bf16(s[j], qa[2 * p + 1][0], qa[2 * p + 1][1], qa[2 * p + 1][2], qa[2 * p + 1][3], b2, b3);
      }
    }
    // ---- online softmax over this block
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const bool valid = (j * 8 + 2 * tq + e) < count;
        s[j][e] = valid ? s[j][e] + beta : -INFINITY;
        s[j][2 + e] = valid ? s[j][2 + e] + beta : -INFINITY;
        mx0 = fmaxf(mx0, s[j][e]);
        mx1 = fmaxf(mx1, s[j][2 + e]);
      }
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
    const float sc0 = v0 ? exp2f((m0 - mn0) * kLog2e) : 1.0f;
    const float sc1 = v1 ? exp2f((m1 - mn1) * kLog2e) : 1.0f;
    m0 = mn0;
    m1 = mn1;
    const float mb0 = mn0 * kLog2e, mb1 = mn1 * kLog2e;
    l0 *= sc0;
    l1 *= sc1;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        s[j][e] = v0 ? exp2f(fmaf(s[j][e], kLog2e, -mb0)) : 0.0f;
        s[j][2 + e] = v1 ? exp2f(fmaf(s[j][2 + e], kLog2e, -mb1)) : 0.0f;
        l0 += s[j][e];
        l1 += s[j][2 + e];
      }
    }
#pragma unroll
    for (int n = 0; n < ON; ++n) {
      o[n][0] *= sc0; o[n][1] *= sc0;
      o[n][2] *= sc1; o[n][3] *= sc1;
    }
    // ---- O += P V  (P re-used from the S accumulators as bf16 A fragments)
#pragma unroll
    for (int kk = 0; kk < NBK / 16; ++kk) {
      const unsigned pa0 = pack_bf16(s[2 * kk][0], s[2 * kk][1]);
      const unsigned pa1 = pack_bf16(s[2 * kk][2], s[2 * kk][3]);
      const unsigned pa2 = pack_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]);
      const unsigned pa3 = pack_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
      for (int np = 0; np < ON / 2; ++np) {
        const int row = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int chunk = np * 2 + (lane >> 4);
        unsigned b0, b1, b2, b3;
        ldsm_x4_t(vbase + row * (DH * 2) + ((chunk ^ (row & 7)) << 4), b0, b1, b2, b3);
        mma_bf16(o[2 * np], pa0, pa1, pa2, pa3, b0, b1);
        mma_bf16(o[2 * np + 1], pa0, pa1, pa2, pa3, b2, b3);
      }
    }
    __syncwarp();
    ++cp_seq;
    ++cp_i;
    advance_loader();  // refill the stage just released

    if (cp_i >= cp_end) {  // end of chunk: write the partial, maybe merge + append
      float lr0 = l0 + __shfl_xor_sync(0xffffffffu, l0, 1);
      lr0 += __shfl_xor_sync(0xffffffffu, lr0, 2);
      float lr1 = l1 + __shfl_xor_sync(0xffffffffu, l1, 1);
      lr1 += __shfl_xor_sync(0xffffffffu, lr1, 2);
      const size_t pbase = (size_t)cp_bh * dv.max_chunks + cp_ci;
      if (v0) {
        float* po = dv.part_o + (pbase * dv.G + g) * DH;
#pragma unroll
        for (int n = 0; n < ON; ++n) *reinterpret_cast<float2*>(po + n * 8 + 2 * tq) = make_float2(o[n][0], o[n][1]);
        if (tq == 0) dv.part_ml[pbase * dv.G + g] = make_float2(m0, lr0);
      }
      if (v1) {
        float* po = dv.part_o + (pbase * dv.G + g + 8) * DH;
#pragma unroll
        for (int n = 0; n < ON; ++n) *reinterpret_cast<float2*>(po + n * 8 + 2 * tq) = make_float2(o[n][2], o[n][3]);
        if (tq == 0) dv.part_ml[pbase * dv.G + g + 8] = make_float2(m1, lr1);
      }
      __threadfence();
      __syncwarp();
      const int nc = (dv.n_req[layer * BH + cp_bh] + kChunk - 1) / kChunk;
      int last = 0;
      if (lane == 0) last = atomicAdd(dv.done + layer * BH + cp_bh, 1) == nc - 1;
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) {
        const int b = cp_bh / dv.H;
        merge_and_append<__nv_bfloat16>(dv, layer, cp_bh, nc, kn, vn, out);
        (void)b;
      }
    }
  }
}

// ---------------------------------------------------------------- fp32 CUDA-core kernel
// Parity path for fp32 storage (tolerance 1e-5): same decomposition, one warp per CTA,
// logits and P.V in fp32 FMA with accurate expf.
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
  int* cbase = reinterpret_cast<int*>(ps + GM * NBK);    // [BH+1]
  int* ring = cbase + BH + 1;                            // [RING]
  int* tmp = ring + RING;                                // [32]
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
      if (lane == 0) c = atomicAdd(dv.cnt + 2 * layer + 1, 1);
      c = __shfl_sync(0xffffffffu, c, 0);
      if (c >= total) { ld_done = true; return; }
      ld_bh = find_bh(cbase, BH, c);
      const int ci = c - cbase[ld_bh];
      ld_i = ci * kChunk;
      ld_end = min(ld_i + kChunk, dv.n_req[layer * BH + ld_bh]);
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
      cp_i = cp_ci * kChunk;
      cp_end = min(cp_i + kChunk, dv.n_req[layer * BH + cp_bh]);
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
    // logits: lane owns keys lane, lane+32, ...
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
        const float p = expf(ps[gg * NBK + key] - mn);
        ps[gg * NBK + key] = p;
        sum += p;
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
        const float p = ps[gg * NBK + key];
#pragma unroll
        for (int x = 0; x < DL; ++x) o[gg][x] = fmaf(p, vv[x], o[gg][x]);
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
        float* po = dv.part_o + (pbase * G + gg) * DH;
#pragma unroll
        for (int x = 0; x < DL; ++x) po[lane + 32 * x] = o[gg][x];
        if (lane == 0) dv.part_ml[pbase * G + gg] = make_float2(m[gg], l[gg]);
      }
      __threadfence();
      __syncwarp();
      const int nc = (dv.n_req[layer * BH + cp_bh] + kChunk - 1) / kChunk;
      int last = 0;
      if (lane == 0) last = atomicAdd(dv.done + layer * BH + cp_bh, 1) == nc - 1;
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) merge_and_append<float>(dv, layer, cp_bh, nc, kn, vn, out);
    }
  }
}

// ---------------------------------------------------------------- launchers
template <int NBK, int DH>
static cudaError_t launch_bf16(const Dev& dv, int layer, const void* q, const void* kn,
                               const void* vn, float* out, cudaStream_t st, int num_sms) {
  constexpr int BPB = 2 * NBK * DH * 2;
  // ~192 KiB of stages per CTA (one CTA per SM): 3 stages per warp, as many warps as fit
  constexpr int NS = 3;
  constexpr int NW = BPB >= 65536 ? 1 : (BPB >= 32768 ? 2 : 4);
  const int BH = dv.B * dv.H;
  const size_t smem = (size_t)NW * NS * BPB + NW * NS * 8 + (BH + 1) * 4 + NW * (NS + 2) * 4 + NW * 32 * 4 + 64;
  auto k = attend_bf16_kernel<NBK, DH, NW, NS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = num_sms;
  k<<<grid, NW * 32, smem, st>>>(dv, layer, static_cast<const __nv_bfloat16*>(q),
                                 static_cast<const __nv_bfloat16*>(kn),
                                 static_cast<const __nv_bfloat16*>(vn), out);
  return cudaGetLastError();
}

template <int NBK, int DH>
static cudaError_t launch_f32(const Dev& dv, int layer, const void* q, const void* kn,
                              const void* vn, float* out, cudaStream_t st, int num_sms) {
  constexpr int NS = 2;
  constexpr int BPB = 2 * NBK * DH * 4;
  const int BH = dv.B * dv.H;
  const size_t smem = (size_t)NS * BPB + NS * 8 + 16 * DH * 4 + 16 * NBK * 4 + (BH + 1) * 4 + (NS + 2) * 4 + 32 * 4 + 64;
  auto k = attend_f32_kernel<NBK, DH, NS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<num_sms, 32, smem, st>>>(dv, layer, static_cast<const float*>(q), static_cast<const float*>(kn),
                               static_cast<const float*>(vn), out);
  return cudaGetLastError();
}

bool attend_supported(int n_b, int d_head, int dtype) {
  const bool nb_ok = n_b == 16 || n_b == 32 || n_b == 64 || n_b == 128;
  const bool d_ok = d_head == 64 || d_head == 128;
  if (dtype == 1 && n_b == 128 && d_head == 128) return false;  // 128 KiB blocks: no double buffer
  return nb_ok && d_ok;
}

cudaError_t launch_attend(const Dev& dv, int layer, const void* q, const void* kn, const void* vn,
                          float* out, cudaStream_t st, int num_sms) {
#define NOSA_DISPATCH(NBK, DH)                                                     \
  if (dv.n_b == NBK && dv.D == DH) {                                               \
    return dv.dtype == 0 ? launch_bf16<NBK, DH>(dv, layer, q, kn, vn, out, st, num_sms) \
                         : launch_f32<NBK, DH>(dv, layer, q, kn, vn, out, st, 2 * num_sms); \
  }
  NOSA_DISPATCH(64, 128)
  NOSA_DISPATCH(64, 64)
  NOSA_DISPATCH(32, 128)
  NOSA_DISPATCH(32, 64)
  NOSA_DISPATCH(16, 128)
  NOSA_DISPATCH(16, 64)
  if (dv.n_b == 128 && dv.D == 64) {
    return dv.dtype == 0 ? launch_bf16<128, 64>(dv, layer, q, kn, vn, out, st, num_sms)
                         : launch_f32<128, 64>(dv, layer, q, kn, vn, out, st, 2 * num_sms);
  }
  if (dv.n_b == 128 && dv.D == 128 && dv.dtype == 0) return launch_bf16<128, 128>(dv, layer, q, kn, vn, out, st, num_sms);
#undef NOSA_DISPATCH
  return cudaErrorInvalidValue;
}

}  // namespace nosa
