// nosa_gather.cu — K3 miss gather (slow -> fast mover) and the prefill / residency-reset
// kernels that set up a run.
//
// K3 is the `mover` of TieredBlockManager.apply_transfers (kv_manager.py:290, 300-305) for the
// whole layer at once: every (lbh, block, slot) entry the planner enqueued is copied from the
// pinned, mapped host mirror into its HBM slot.  The SMs read host memory directly over PCIe
// (zero-copy UVA), so the copy needs no host round trip to learn the miss list.
#include <cstdlib>

#include "nosa_device.cuh"

namespace nosa {

// grid = a few dozen CTAs (latency-bound on PCIe, leaves SMs to the attention kernel)
// 16-byte load from pinned host memory; with L2HINT the L2 fetches whole 256-byte lines
// (ld.global.nc.L2::256B), so the PCIe read requests are larger.
template <bool L2HINT>
__device__ __forceinline__ int4 ld_host(const int4* p) {
  if constexpr (L2HINT) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
  } else {
    return __ldcs(p);
  }
}

// Each CTA copies NBLK list entries per iteration: NBLK * bpb / (256 * 16) 16-byte loads per
// thread are issued before any store, so NBLK * 32 KiB per CTA are in flight on the link.
// One grid walks the layers [layer0, layer0 + nl) in order, so the SM loads in flight over PCIe
// do not grow with the layers of an attention batch: zero-copy reads are served through L2, and
// more than ~8 CTAs of them slow the attention's HBM stream and the link itself (measured,
// tools/mover_probe.cu: an HBM stream keeps 0.91x of its rate next to 8 CTAs, 0.60x next to 32).
template <int NBLK, bool L2HINT>
__global__ void __launch_bounds__(256) gather_kernel(Dev dv, int layer0, int nl) {
  constexpr int PER = 8;  // 16-byte vectors per thread per 32 KiB block at 256 threads
  const int vecs = (int)(dv.bpb / 16);
  for (int layer = layer0; layer < layer0 + nl; ++layer) {
    const int n = *reinterpret_cast<volatile int*>(dv.cnt + kCntStride * layer);
    const int4* list = dv.miss_list + (size_t)layer * dv.B * dv.H * dv.C;
    for (int e0 = blockIdx.x * NBLK; e0 < n; e0 += gridDim.x * NBLK) {
      int4 m[NBLK];
#pragma unroll
      for (int j = 0; j < NBLK; ++j) m[j] = e0 + j < n ? list[e0 + j] : make_int4(-1, 0, 0, 0);
      for (int base = threadIdx.x; base < vecs; base += blockDim.x * PER) {
        int4 v[NBLK][PER];
#pragma unroll
        for (int j = 0; j < NBLK; ++j) {
          if (m[j].x < 0 || m[j].w) continue;
          const int4* src = reinterpret_cast<const int4*>(dv.host + ((size_t)m[j].x * dv.NB + m[j].y) * dv.bpb);
#pragma unroll
          for (int u = 0; u < PER; ++u) {
            const int i = base + u * blockDim.x;
            if (i < vecs) v[j][u] = ld_host<L2HINT>(src + i);
          }
        }
#pragma unroll
        for (int j = 0; j < NBLK; ++j) {
          if (m[j].x < 0 || m[j].w) continue;
          int4* dst = reinterpret_cast<int4*>(dv.pool + ((size_t)m[j].x * dv.C + m[j].z) * dv.bpb);
#pragma unroll
          for (int u = 0; u < PER; ++u) {
            const int i = base + u * blockDim.x;
            if (i < vecs) dst[i] = v[j][u];
          }
        }
      }
#pragma unroll
      for (int j = 0; j < NBLK; ++j)
        if (m[j].x >= 0 && m[j].w == 1)  // (w = 2: moved by the host-pack path)
          write_born_block(dv, m[j], reinterpret_cast<int4*>(dv.pool + ((size_t)m[j].x * dv.C + m[j].z) * dv.bpb), vecs);
    }
  }
}

// TMA variant: one warp per CTA streams blocks host -> shared (cp.async.bulk, mbarrier) ->
// HBM slot (cp.async.bulk shared -> global, bulk groups) through a ring of stages, so the PCIe
// reads are issued by the TMA engine in large requests instead of 16-byte SM loads.
constexpr int kTmaStages = 4;

__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__global__ void __launch_bounds__(32) gather_tma_kernel(Dev dv, int layer0, int nl) {
  extern __shared__ __align__(128) char smem_raw[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + (size_t)kTmaStages * dv.bpb);
  const int lane = threadIdx.x;
  if (lane == 0) {
    for (int s = 0; s < kTmaStages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  int k_base = 0;  // items issued by this CTA in earlier layers: the ring's stage and phase run on
  for (int layer = layer0; layer < layer0 + nl; ++layer) {
    const int n = *reinterpret_cast<volatile int*>(dv.cnt + kCntStride * layer);
    const int4* list = dv.miss_list + (size_t)layer * dv.B * dv.H * dv.C;
    const int m = n > (int)blockIdx.x ? (n - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;  // items of this CTA
    auto item = [&](int k) { return list[blockIdx.x + (size_t)k * gridDim.x]; };
    auto issue = [&](int k) {  // host -> stage (born blocks are written directly, see below)
      const int4 e = item(k);
      const int s = (k_base + k) % kTmaStages;
      if (e.w) {  // born (rebuilt below) or moved by the host-pack path: nothing to load
        mbar_arrive_plain(&bars[s]);
        return;
      }
      mbar_expect_tx(&bars[s], (unsigned)dv.bpb);
      bulk_g2s(smem_raw + (size_t)s * dv.bpb, dv.host + ((size_t)e.x * dv.NB + e.y) * dv.bpb, (unsigned)dv.bpb, &bars[s]);
    };
    if (lane == 0)
      for (int k = 0; k < min(kTmaStages, m); ++k) issue(k);
    for (int k = 0; k < m; ++k) {
      const int s = (k_base + k) % kTmaStages;
      const int4 e = item(k);
      char* dst = dv.pool + ((size_t)e.x * dv.C + e.z) * dv.bpb;
      mbar_wait(&bars[s], ((k_base + k) / kTmaStages) & 1);
      if (e.w == 1) {  // born at the previous step: row 0 from the device stash, zeros elsewhere
        const int vecs = (int)(dv.bpb / 16), row_vecs = dv.D * dv.elem / 16, plane_vecs = vecs / 2;
        const int4* stash = reinterpret_cast<const int4*>(dv.newrow + (size_t)e.x * 2 * dv.D * dv.elem);
        for (int i = lane; i < vecs; i += 32) {
          const int which = i / plane_vecs, in_plane = i - which * plane_vecs;
          reinterpret_cast<int4*>(dst)[i] = in_plane < row_vecs ? stash[which * row_vecs + in_plane] : make_int4(0, 0, 0, 0);
        }
        __syncwarp();
      } else if (e.w == 0 && lane == 0) {
        bulk_s2g(dst, smem_raw + (size_t)s * dv.bpb, (unsigned)dv.bpb);
        bulk_commit();
      }
      if (lane == 0 && k + kTmaStages < m) {
        bulk_wait_read_all();  // the store has finished reading stage s
        issue(k + kTmaStages);
      }
    }
    if (lane == 0) bulk_wait_all();  // the ring is reused by the next layer
    __syncwarp();
    k_base += m;
  }
}

// Blocks born by the previous step's append, for the copy-engine mover: the memcpy batch skips
// them (their only valid row is in the device stash), this kernel writes them into their slots.
__global__ void __launch_bounds__(256) born_kernel(Dev dv, int layer) {
  const int n = dv.cnt[kCntStride * layer];
  const int4* list = dv.miss_list + (size_t)layer * dv.B * dv.H * dv.C;
  const int vecs = (int)(dv.bpb / 16);
  for (int e = blockIdx.x; e < n; e += gridDim.x) {
    const int4 m = list[e];
    if (m.w == 1) write_born_block(dv, m, reinterpret_cast<int4*>(dv.pool + ((size_t)m.x * dv.C + m.z) * dv.bpb), vecs);
  }
}

// Host-pack mover: one DMA'd chunk of packed blocks, device ring -> their slots (HBM -> HBM).
__global__ void __launch_bounds__(256) scatter_kernel(const int4* __restrict__ stage, void* const* __restrict__ dst,
                                                      int count, int vecs) {
  for (int e = blockIdx.x; e < count; e += gridDim.x) {
    const int4* s = stage + (size_t)e * vecs;
    int4* d = reinterpret_cast<int4*>(dst[e]);
    for (int i = threadIdx.x; i < vecs; i += blockDim.x) d[i] = __ldcs(s + i);
  }
}

cudaError_t launch_scatter(const char* stage, void* const* dst, int count, int bpb, cudaStream_t st) {
  scatter_kernel<<<count, 256, 0, st>>>(reinterpret_cast<const int4*>(stage), dst, count, bpb / 16);
  return cudaGetLastError();
}

cudaError_t launch_born(const Dev& dv, int layer, cudaStream_t st, int grid) {
  born_kernel<<<grid, 256, 0, st>>>(dv, layer);
  return cudaGetLastError();
}

// layers [layer, layer + nl) in one launch
cudaError_t launch_gather(const Dev& dv, int layer, cudaStream_t st, int grid, bool tma, int nl) {
  const dim3 g(grid);
  if (tma) {
    const size_t smem = (size_t)kTmaStages * dv.bpb + kTmaStages * 8;
    cudaFuncSetAttribute(gather_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    max_shared_carveout(gather_tma_kernel);
    gather_tma_kernel<<<g, 32, smem, st>>>(dv, layer, nl);
  } else {
    // NOSA_GATHER_VARIANT: bit 0 = two blocks per CTA iteration, bit 1 = L2::256B.  Default 2
    // for 32 KiB blocks: the 256-byte L2 fetch hint (cfg 3, two alternations: 14.13K vs 13.97K
    // tok/s, attention next to the gather 0.83 vs 0.77 of HBM; tools/r2u.sh).  Default 3 for
    // larger (fp32) blocks, which take two 32 KiB passes each: two blocks per iteration keep
    // 64 KiB per CTA in flight (cfg 3 fp32 with 12 CTAs: 6.36K vs 5.13K tok/s; tools/r2bb.sh)
    static const int env_variant = getenv("NOSA_GATHER_VARIANT") ? atoi(getenv("NOSA_GATHER_VARIANT")) : -1;
    const int variant = env_variant >= 0 ? env_variant : (dv.bpb > 32768 ? 3 : 2);
    max_shared_carveout(gather_kernel<1, false>);
    max_shared_carveout(gather_kernel<2, false>);
    max_shared_carveout(gather_kernel<1, true>);
    max_shared_carveout(gather_kernel<2, true>);
    switch (variant & 3) {
      case 0: gather_kernel<1, false><<<g, 256, 0, st>>>(dv, layer, nl); break;
      case 1: gather_kernel<2, false><<<g, 256, 0, st>>>(dv, layer, nl); break;
      case 2: gather_kernel<1, true><<<g, 256, 0, st>>>(dv, layer, nl); break;
      default: gather_kernel<2, true><<<g, 256, 0, st>>>(dv, layer, nl); break;
    }
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// Input staging of nosa_decode_step_host: up to three host segments (q, k_new, v_new of a
// selection group) copied into device memory by the SMs with zero-copy 16-byte loads from the
// mapped pinned buffers.  The copy engine is busy with the miss gathers and runs its queue in
// order; SM loads share the PCIe link with it instead of queueing behind it.
__global__ void __launch_bounds__(256) stage_inputs_kernel(StageSeg a, StageSeg b, StageSeg c) {
  constexpr int PER = 4;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (const StageSeg& sg : {a, b, c}) {
    for (long long i0 = tid; i0 < sg.n16; i0 += stride * PER) {
      int4 v[PER];
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const long long i = i0 + u * stride;
        if (i < sg.n16) v[u] = ld_host<true>(sg.src + i);  // 256-byte L2 fetches, like the gather
      }
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const long long i = i0 + u * stride;
        if (i < sg.n16) sg.dst[i] = v[u];
      }
    }
  }
}

const void* stage_inputs_kernel_fn() { return reinterpret_cast<const void*>(stage_inputs_kernel); }

cudaError_t launch_stage_inputs(const void* const* src, void* const* dst, const size_t* bytes, int grid,
                                cudaStream_t st) {
  StageSeg sg[3];
  for (int i = 0; i < 3; ++i)
    sg[i] = {static_cast<const int4*>(src[i]), static_cast<int4*>(dst[i]), (long long)(bytes[i] / 16)};
  max_shared_carveout(stage_inputs_kernel);
  stage_inputs_kernel<<<grid, 256, 0, st>>>(sg[0], sg[1], sg[2]);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// Prefill, step 1: K/V rows [S][H][t][D] -> swizzled block format [S*H][NB][2][n_b][D] in a
// device staging buffer (zero padded past t), later copied to the host mirror in one DMA.
template <typename T>
__global__ void __launch_bounds__(256) prefill_layout_kernel(Dev dv, const T* __restrict__ k, const T* __restrict__ v,
                                                             int t, int S, char* __restrict__ staging) {
  // one CTA per (s*h, block), grid-striding: a block's K rows (and V rows) are n_b contiguous
  // rows of the input, read as 16-byte chunks and written swizzled into its 32 KiB slot image
  const int elem = sizeof(T);
  const int D = dv.D, n_b = dv.n_b;
  const int cpr = D * elem / 16;           // 16-byte chunks per row
  const int per_plane = n_b * cpr;
  const int total = S * dv.H * dv.NB;
  for (int g = blockIdx.x; g < total; g += gridDim.x) {
    const int sh = g / dv.NB, blk = g - sh * dv.NB;
    const int lo = blk * n_b;
    char* dst_blk = staging + (size_t)g * dv.bpb;
    for (int c = threadIdx.x; c < 2 * per_plane; c += blockDim.x) {
      const int which = c >= per_plane, rem = c - which * per_plane;
      const int row = rem / cpr, ch = rem - row * cpr;
      const int tok = lo + row;
      int4 val = make_int4(0, 0, 0, 0);
      if (tok < t) val = reinterpret_cast<const int4*>((which ? v : k) + ((size_t)sh * t + tok) * D)[ch];
      *reinterpret_cast<int4*>(dst_blk + (size_t)which * n_b * D * elem + (size_t)row * D * elem +
                               ((ch ^ (row & 7)) << 4)) = val;
    }
  }
}

// Prefill, step 2: per block of the prefix, the f64 block means of K (compress_blocks,
// attention.py:42-59) and of the per-token importance scores (importance_scores +
// compress_scores, attention.py:62-64, 121-146); partial tail block -> running sums.
// One warp per (s, h, block).
template <typename T>
__global__ void prefill_stats_kernel(Dev dv, int layer, int seq_begin, const T* __restrict__ k,
                                     const T* __restrict__ v, int t, int S) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nblk = (t + dv.n_b - 1) / dv.n_b;
  const int total = S * dv.H * nblk;
  if (gw >= total) return;
  const int sh = gw / nblk, blk = gw - sh * nblk;
  const int s = sh / dv.H, h = sh - s * dv.H;
  const int lbh = (layer * dv.B + seq_begin + s) * dv.H + h;
  const int D = dv.D, n_b = dv.n_b;
  const int lo = blk * n_b, cnt = min(n_b, t - lo);
  double se_sum = 0.0;
  double ks[8];  // D <= 256
#pragma unroll
  for (int j = 0; j < 8; ++j) ks[j] = 0.0;
  for (int r = 0; r < cnt; ++r) {
    const T* krow = k + ((size_t)sh * t + lo + r) * D;
    const T* vrow = v + ((size_t)sh * t + lo + r) * D;
    se_sum += token_score_warp<T>(vrow, dv.w1, dv.w2, D, dv.n_ev, dv.variant);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int d = lane + 32 * j;
      if (d < D) ks[j] += to_f64(krow[d]);
    }
  }
  if (cnt == n_b) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int d = lane + 32 * j;
      if (d < D) dv.kc[((size_t)lbh * dv.NB + blk) * D + d] = ks[j] / (double)n_b;
    }
    if (lane == 0) dv.se[(size_t)lbh * dv.NB + blk] = se_sum / (double)n_b;
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int d = lane + 32 * j;
      if (d < D) dv.tail_ksum[(size_t)lbh * D + d] = ks[j];
    }
    if (lane == 0) dv.tail_se[lbh] = se_sum;
  }
}

// Prefill, step 2 (the path used): one CTA of 256 threads per (s, h, block), grid-striding over
// blocks.  One pass over the block loads its V rows into shared memory (fp32, padded rows) and
// sums K per column in registers.  The importance scores of the block's tokens are one small
// fp64 GEMM, Z[n_b][n_ev] = V[n_b][D] . W1[D][n_ev], on the FP64 tensor cores
// (mma.m8n8k4.f64: warp w owns 8-token tiles, W1 pre-arranged per lane as B fragments), then
// silu(Z) . W2 per token from the accumulator fragments.  Every sum has a fixed order
// (deterministic); the K sums are exact in f64 for bf16 / fp32 rows.  Measured on one cfg 3
// layer (B=128, 32K, ncu): 10.2 ms against 117 ms for prefill_stats_kernel.
__device__ __forceinline__ void dmma_m8n8k4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

constexpr int kPrefillNT = 4;  // up to 32 eviction-head columns (n-tiles of 8)

template <typename T>
__global__ void __launch_bounds__(256) prefill_block_kernel(Dev dv, int layer, int seq_begin, const T* __restrict__ k,
                                                            const T* __restrict__ v, int t, int S) {
  extern __shared__ __align__(16) char smem[];
  const int D = dv.D, n_b = dv.n_b, n_ev = dv.n_ev, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NT = (n_ev + 7) / 8, KS = D / 4, VLD = D + 4;
  double* w1f = reinterpret_cast<double*>(smem);         // [KS][NT][32] B fragments
  double* red = w1f + (size_t)KS * NT * 32;               // [256] K partials, then token scores
  float* vt = reinterpret_cast<float*>(red + 256);        // [n_b][D + 4]
  for (int x = tid; x < KS * NT * 32; x += blockDim.x) {  // lane (k = lane % 4, n = lane / 4)
    const int l = x & 31, f = x >> 5, nt = f % NT, ks = f / NT;
    const int i = 4 * ks + (l & 3), j = 8 * nt + (l >> 2);
    w1f[x] = j < n_ev ? dv.w1[(size_t)i * n_ev + j] : 0.0;
  }
  const int nblk = (t + n_b - 1) / n_b;
  const int total = S * dv.H * nblk;
  for (int g = blockIdx.x; g < total; g += gridDim.x) {
    const int sh = g / nblk, blk = g - sh * nblk;
    const int s = sh / dv.H, h = sh - s * dv.H;
    const int lbh = (layer * dv.B + seq_begin + s) * dv.H + h;
    const int lo = blk * n_b, cnt = min(n_b, t - lo);
    const T* kb = k + ((size_t)sh * t + lo) * D;
    const T* vb = v + ((size_t)sh * t + lo) * D;
    __syncthreads();  // W1 staged / the previous block's tile and scores consumed
    // one pass over the tile: V rows into shared memory, K column partial sums in registers
    // (D divides the CTA: thread tid always sees column tid % D; every load independent)
    double kpart = 0.0;
#pragma unroll 4
    for (int x = tid; x < cnt * D; x += blockDim.x) {
      const int r = x / D, i = x - r * D;
      vt[r * VLD + i] = (float)to_f64(vb[x]);
      kpart += to_f64(kb[x]);
    }
    red[tid] = kpart;
    __syncthreads();
    if (tid < D) {  // K block sums
      double ks = 0.0;
      for (int u = tid; u < (int)blockDim.x; u += D) ks += red[u];
      if (cnt == n_b) dv.kc[((size_t)lbh * dv.NB + blk) * D + tid] = ks / (double)n_b;
      else dv.tail_ksum[(size_t)lbh * D + tid] = ks;
    }
    __syncthreads();
    // token scores: 8-token tiles on the FP64 tensor cores (rows past cnt read stale shared
    // memory; MMA rows are independent and theirs are dropped)
    for (int mt = warp; mt < n_b / 8; mt += blockDim.x / 32) {
      double acc[kPrefillNT][2];
#pragma unroll
      for (int nt = 0; nt < kPrefillNT; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
      const float* arow = vt + (8 * mt + (lane >> 2)) * VLD + (lane & 3);
      for (int ks = 0; ks < KS; ++ks) {
        const double a = (double)arow[4 * ks];
        const double* bf = w1f + (size_t)ks * NT * 32 + lane;
#pragma unroll
        for (int nt = 0; nt < kPrefillNT; ++nt)
          if (nt < NT) dmma_m8n8k4(acc[nt], a, bf[nt * 32]);
      }
      // lane holds Z[token 8 mt + lane / 4][columns 8 nt + 2 (lane % 4) + {0, 1}]
      double part = 0.0;
#pragma unroll
      for (int nt = 0; nt < kPrefillNT; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int j = 8 * nt + 2 * (lane & 3) + e;
          if (nt < NT && j < n_ev) part = fma(silu64(acc[nt][e]), dv.w2[j], part);
        }
      part += __shfl_xor_sync(0xffffffffu, part, 1);
      part += __shfl_xor_sync(0xffffffffu, part, 2);
      const int tok = 8 * mt + (lane >> 2);
      if ((lane & 3) == 0 && tok < cnt) red[tok] = dv.variant == 2 ? exp(part) : part;
    }
    __syncthreads();
    if (tid == 0) {
      double se = 0.0;
      for (int rr = 0; rr < cnt; ++rr) se += red[rr];
      if (cnt == n_b) dv.se[(size_t)lbh * dv.NB + blk] = se / (double)n_b;
      else dv.tail_se[lbh] = se;
    }
  }
}

// Reset the residency of [seq_begin, seq_begin+S) in one layer: every block slow-resident,
// fresh LIFO free lists (kv_manager.py:147-150), cache length t.
__global__ void reset_residency_kernel(Dev dv, int layer, int seq_begin, int S, int t) {
  const int sh = blockIdx.x;
  const int lbh = (layer * dv.B + seq_begin) * dv.H + sh;  // S*H consecutive lbh
  for (int i = threadIdx.x; i < dv.NB; i += blockDim.x) dv.slot_of[(size_t)lbh * dv.NB + i] = -1;
  // shared pool: this row holds entries [b*C, b*C + C) of the layer-head's B*C-slot free stack
  const int b = seq_begin + sh / dv.H;
  const int n_free = dv.shared ? dv.B * dv.C : dv.C;
  const int first = dv.shared ? b * dv.C : 0;
  for (int i = threadIdx.x; i < dv.C; i += blockDim.x) {
    dv.blk_of[(size_t)lbh * dv.C + i] = -1;
    dv.lastreq[(size_t)lbh * dv.C + i] = 0;
    dv.fstack[(size_t)lbh * dv.C + i] = n_free - 1 - (first + i);
  }
  if (threadIdx.x == 0) {
    dv.ftop[lbh] = n_free;
    dv.clock[lbh] = 0;
    dv.t[lbh] = t;
    dv.t0[lbh] = t;
    dv.n_req[lbh] = 0;
    if (t % dv.n_b == 0) {
      dv.tail_se[lbh] = 0.0;
    }
  }
  if (t % dv.n_b == 0)
    for (int d = threadIdx.x; d < dv.D; d += blockDim.x) dv.tail_ksum[(size_t)lbh * dv.D + d] = 0.0;
}

// Blocks [0, nblk) of S consecutive sequences become fast-resident in slots [0, nblk):
// block i -> slot i, free stack holds [C-1 .. nblk] (what nblk LIFO pops leave behind).
__global__ void make_resident_kernel(Dev dv, int layer, int seq_begin, int nblk) {
  const int lbh = (layer * dv.B + seq_begin) * dv.H + blockIdx.x;
  for (int i = threadIdx.x; i < dv.C; i += blockDim.x) {
    dv.blk_of[(size_t)lbh * dv.C + i] = i < nblk ? i : -1;
    dv.lastreq[(size_t)lbh * dv.C + i] = 0;
    dv.fstack[(size_t)lbh * dv.C + i] = dv.C - 1 - i;
  }
  for (int i = threadIdx.x; i < dv.NB; i += blockDim.x) dv.slot_of[(size_t)lbh * dv.NB + i] = i < nblk ? i : -1;
  if (threadIdx.x == 0) dv.ftop[lbh] = dv.C - nblk;
}

cudaError_t launch_make_resident(const Dev& dv, int layer, int seq_begin, int S, int nblk, cudaStream_t st) {
  make_resident_kernel<<<S * dv.H, 256, 0, st>>>(dv, layer, seq_begin, nblk);
  return cudaGetLastError();
}

cudaError_t launch_prefill(const Dev& dv, int layer, int seq_begin, int S, const void* k,
                           const void* v, int t, char* staging, cudaStream_t st) {
  const int nblk = (t + dv.n_b - 1) / dv.n_b;
  reset_residency_kernel<<<S * dv.H, 256, 0, st>>>(dv, layer, seq_begin, S, t);
  const int warps = S * dv.H * nblk;
  const int blocks = (warps * 32 + 255) / 256;
  // block kernel: n_b % 8 == 0, D divides 256, n_ev <= 32 (every supported shape);
  // NOSA_PREFILL_WARP=1 keeps the warp-per-block kernel (experiments)
  const size_t bsmem = (size_t)(dv.D / 4) * ((dv.n_ev + 7) / 8) * 32 * 8 + 256 * 8 + (size_t)dv.n_b * (dv.D + 4) * 4;
  static const bool warp_env = getenv("NOSA_PREFILL_WARP") != nullptr;
  const bool block_ok = !warp_env && dv.n_b % 8 == 0 && dv.n_b <= 256 && 256 % dv.D == 0 && dv.D % 4 == 0 &&
                        dv.n_ev <= 8 * kPrefillNT && bsmem <= 200 * 1024;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int bgrid = std::max(1, std::min(warps, sms * 4));
  if (dv.dtype == 0) {
    prefill_layout_kernel<__nv_bfloat16><<<sms * 8, 256, 0, st>>>(
        dv, static_cast<const __nv_bfloat16*>(k), static_cast<const __nv_bfloat16*>(v), t, S, staging);
    if (warps > 0 && block_ok) {
      max_shared_carveout(prefill_block_kernel<__nv_bfloat16>);
      cudaFuncSetAttribute(prefill_block_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsmem);
      prefill_block_kernel<__nv_bfloat16><<<bgrid, 256, bsmem, st>>>(dv, layer, seq_begin,
                                                                      static_cast<const __nv_bfloat16*>(k),
                                                                      static_cast<const __nv_bfloat16*>(v), t, S);
    } else if (warps > 0) {
      prefill_stats_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>(
          dv, layer, seq_begin, static_cast<const __nv_bfloat16*>(k),
          static_cast<const __nv_bfloat16*>(v), t, S);
    }
  } else {
    prefill_layout_kernel<float><<<sms * 8, 256, 0, st>>>(dv, static_cast<const float*>(k),
                                                       static_cast<const float*>(v), t, S, staging);
    if (warps > 0 && block_ok) {
      max_shared_carveout(prefill_block_kernel<float>);
      cudaFuncSetAttribute(prefill_block_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsmem);
      prefill_block_kernel<float><<<bgrid, 256, bsmem, st>>>(dv, layer, seq_begin, static_cast<const float*>(k),
                                                            static_cast<const float*>(v), t, S);
    } else if (warps > 0) {
      prefill_stats_kernel<float><<<blocks, 256, 0, st>>>(dv, layer, seq_begin, static_cast<const float*>(k),
                                                          static_cast<const float*>(v), t, S);
    }
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// Readback helper: un-swizzle n blocks [n][2][n_b][D] (storage format) into [2][n][n_b][D]
// row order (K rows then V rows), on the device.
__global__ void unswizzle_kernel(const char* __restrict__ src, char* __restrict__ dst, int nblocks,
                                 int n_b, int D, int elem) {
  const int chunks_per_row = D * elem / 16;
  const long long total = (long long)nblocks * 2 * n_b * chunks_per_row;
  for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < total;
       x += (long long)gridDim.x * blockDim.x) {
    const int ch = (int)(x % chunks_per_row);
    const long long rr = x / chunks_per_row;  // (blk, which, row)
    const int row = (int)(rr % n_b);
    const long long bw = rr / n_b;
    const int which = (int)(bw % 2);
    const long long blk = bw / 2;
    const int4 val = *reinterpret_cast<const int4*>(src + (size_t)rr * D * elem + ((ch ^ (row & 7)) << 4));
    char* o = dst + (((size_t)which * nblocks + blk) * n_b + row) * D * elem + (size_t)ch * 16;
    *reinterpret_cast<int4*>(o) = val;
  }
}

cudaError_t launch_unswizzle(const char* src, char* dst, int nblocks, int n_b, int D, int elem,
                             cudaStream_t st) {
  unswizzle_kernel<<<256, 256, 0, st>>>(src, dst, nblocks, n_b, D, elem);
  return cudaGetLastError();
}

}  // namespace nosa
