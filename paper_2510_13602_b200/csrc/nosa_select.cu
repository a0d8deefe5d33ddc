// nosa_select.cu — K1 (block selection) and K2 (GPU-resident block-cache planner).
//
// K1 restates, per (sequence, kv head), the selection half of DecodeEngine.step
// (decode.py:169-176): GQA-summed query scoring of the frozen pool (decode.py:171-172),
// then nosa_select (selection.py:130-160) or infllmv2_select (selection.py:163-178) with
// argtopk's order (numerics.py:59-73: score desc, index asc).  Scores are computed in f64
// from f64 block means so the chosen sets agree with the f64 oracle except on exact ties.
// K2 restates TieredBlockManager.plan_transfers + apply_transfers (kv_manager.py:205-298)
// for one manager per (sequence, kv head): hit test, least-recently-required victims
// (kv_manager.py:125-127), LIFO free-slot reuse (kv_manager.py:147-150, 281-298).
#include "nosa_device.cuh"

namespace nosa {

// Bitonic sort of Pp (power of two) (key, idx) pairs in shared memory, best first:
// larger key wins, equal keys -> smaller idx wins.  Called by the whole block.
__device__ void block_sort_best_first(unsigned long long* key, int* idx, int Pp) {
  for (int k = 2; k <= Pp; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < Pp; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const unsigned long long ka = key[i], kb = key[ixj];
          const int ia = idx[i], ib = idx[ixj];
          const bool b_better = (kb > ka) || (kb == ka && ib < ia);
          const bool a_better = (ka > kb) || (ka == kb && ia < ib);
          const bool up = (i & k) == 0;
          if (up ? b_better : a_better) {
            key[i] = kb; key[ixj] = ka;
            idx[i] = ib; idx[ixj] = ia;
          }
        }
      }
      __syncthreads();
    }
  }
}

__device__ __forceinline__ int next_pow2(int x) {
  int p = 32;
  while (p < x) p <<= 1;
  return p;
}

// Writes the ascending list of set bits of bm (nwords words, bit p -> value base + p) to out.
// One warp.  Returns the count.
__device__ int warp_bits_to_sorted(const unsigned* bm, int nwords, int base, int* out) {
  const int lane = threadIdx.x & 31;
  int n = 0;
  for (int w = 0; w < nwords; ++w) {
    const unsigned word = bm[w];
    if (word == 0u) continue;
    const bool set = (word >> lane) & 1u;
    if (set) out[n + __popc(word & ((1u << lane) - 1u))] = base + w * 32 + lane;
    n += __popc(word);
  }
  return n;
}

struct SelSmem {
  double* qsum;
  unsigned long long* key;
  int* idx;
  unsigned* bm_q;
  unsigned* bm_e;
  int* req;
  int* reqslot;
  int* fetch;
  int* fpos;
  int* victims;
  unsigned long long* ckey;
  unsigned* lo_key;  // [Pp] screened lower bound of each pool row (monotone u32 of the float)
  float* up;         // [Pp] screened upper bound
  int* hist;         // [256] radix-select histogram
  int* misc;  // [16]
  long long* marks;  // diagnostics: clock64 at phase boundaries (NULL = off)
};

__device__ SelSmem carve_sel_smem(char* base, int D, int Pp, int C) {
  SelSmem s;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* p = base + off;
    off += (bytes + 15) & ~size_t(15);
    return p;
  };
  s.qsum = reinterpret_cast<double*>(take(sizeof(double) * D));
  s.key = reinterpret_cast<unsigned long long*>(take(sizeof(unsigned long long) * Pp));
  s.idx = reinterpret_cast<int*>(take(sizeof(int) * Pp));
  s.bm_q = reinterpret_cast<unsigned*>(take(sizeof(unsigned) * (Pp / 32)));
  s.bm_e = reinterpret_cast<unsigned*>(take(sizeof(unsigned) * (Pp / 32)));
  s.req = reinterpret_cast<int*>(take(sizeof(int) * C));
  s.reqslot = reinterpret_cast<int*>(take(sizeof(int) * C));
  s.fetch = reinterpret_cast<int*>(take(sizeof(int) * C));
  s.fpos = reinterpret_cast<int*>(take(sizeof(int) * C));
  s.victims = reinterpret_cast<int*>(take(sizeof(int) * C));
  s.ckey = reinterpret_cast<unsigned long long*>(take(sizeof(unsigned long long) * C));
  s.lo_key = reinterpret_cast<unsigned*>(take(sizeof(unsigned) * Pp));
  s.up = reinterpret_cast<float*>(take(sizeof(float) * Pp));
  s.hist = reinterpret_cast<int*>(take(sizeof(int) * 256));
  s.misc = reinterpret_cast<int*>(take(sizeof(int) * 16));
  return s;
}

size_t sel_smem_bytes(int D, int Pp, int C) {
  auto r = [](size_t b) { return (b + 15) & ~size_t(15); };
  return r(8 * D) + r(8 * (size_t)Pp) + r(4 * (size_t)Pp) + 2 * r(4 * (size_t)(Pp / 32)) +
         5 * r(4 * (size_t)C) + r(8 * (size_t)C) + 2 * r(4 * (size_t)Pp) + r(4 * 256) + r(64);
}

enum { M_NREQ = 0, M_NF, M_SHORT, M_NCAND, M_CLOCK, M_ERR, M_NQ, M_NE, M_QMAX, M_BIN, M_REM, M_NC };

// diagnostics (Dev.sel_prof): phase boundary i of this CTA
__device__ __forceinline__ void sel_mark(const SelSmem& sm, int i) {
  if (sm.marks && threadIdx.x == 0) sm.marks[i] = clock64();
}

// monotone u32 image of a float (larger float -> larger key), and back
__device__ __forceinline__ unsigned f2key(float f) {
  const unsigned b = __float_as_uint(f == 0.0f ? 0.0f : f);
  return (b >> 31) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float key2f(unsigned k) {
  return __uint_as_float((k >> 31) ? (k & 0x7fffffffu) : ~k);
}

// f64 dot of one K_c row with q_sum by one warp, every lane ends with the sum.  The screened
// selector's refinement and the parity readback of s_q both use exactly this order.
__device__ __forceinline__ double row_dot64(const double* __restrict__ row, const double* qs, int D) {
  const int lane = threadIdx.x & 31;
  double a = 0.0;
  for (int i = lane * 2; i < D; i += 64) {
    const double2 v = __ldg(reinterpret_cast<const double2*>(row + i));
    a = fma(v.y, qs[i + 1], fma(v.x, qs[i], a));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  return a;
}

// Exact top-m of the pool by s_q = K_c . q_sum (f64), from a bf16 pre-scan.  Every pool row
// gets an interval [lo, up] that provably contains its f64 score: the bf16 dot in fp32 plus
// (fp32 accumulation bound) + (rounding of K_c to bf16: sum|K_c - bf16(K_c)| * max|q_sum|) +
// (rounding of q_sum to fp32) + (f64 accumulation bound).  T = the m-th largest lower bound
// (radix select); a row with up < T has m rows strictly above it, so only rows with up >= T
// are candidates, rescored in f64 and ranked by (score desc, index asc) = argtopk's order.
// Sets the picked bits in sm.bm_q.  bf16 rows are 4x fewer bytes than the f64 scan.
// (a) screen of pool rows [pb, pe): a half-warp per row (16 lanes x D/16 dims: one 16-byte load
//     per lane at D=128), 16 rows per warp iteration with every load issued first, then a
//     reduce-scatter over the 16 lanes leaves row u's dot and abs-dot on lane 2*u' (u' =
//     bit-reversed position).  Writes each row's interval [lo, up] (lo as a monotone key) to
//     lo_out / up_out (shared memory when fused, the global scratch when split).
// loads of one warp iteration of (a): rows p0 + 2u + half, lane hl's 16-byte slice
// (+ the K_c rounding bound of the row this lane will write, so it is in flight with the rows)
__device__ __forceinline__ void screen_load(const __nv_bfloat16* __restrict__ k16, const float* __restrict__ kerr,
                                            int D, int p0, int pe, uint4 (&raw)[8], float& kr) {
  const int lane = threadIdx.x & 31, hl = lane & 15, half = lane >> 4, E = D / 16;
  kr = __ldg(kerr + min(p0 + 2 * (((hl & 8) ? 4 : 0) + ((hl & 4) ? 2 : 0) + ((hl & 2) ? 1 : 0)) + half, pe - 1));
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const __nv_bfloat16* row = k16 + (size_t)min(p0 + 2 * u + half, pe - 1) * D + hl * E;
    if (E == 8) {
      raw[u] = __ldg(reinterpret_cast<const uint4*>(row));
    } else {
      const uint2 r2 = __ldg(reinterpret_cast<const uint2*>(row));
      raw[u] = make_uint4(r2.x, r2.y, 0u, 0u);
    }
  }
}

// the rest of (a) for one warp iteration: dots, the 16-lane reduce-scatter, the intervals
__device__ __forceinline__ void screen_finish(const uint4 (&raw)[8], const float (&qf)[8], float kr,
                                             float gam, float qmax, int p0, int pe, unsigned* lo_out,
                                             float* up_out) {
  const int lane = threadIdx.x & 31, hl = lane & 15, half = lane >> 4;
  float sv[8], av[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const unsigned w[4] = {raw[u].x, raw[u].y, raw[u].z, raw[u].w};
    float sacc = 0.0f, aacc = 0.0f;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const __nv_bfloat162 x = *reinterpret_cast<const __nv_bfloat162*>(&w[j]);
      const float k0 = __low2float(x), k1 = __high2float(x);
      sacc = fmaf(k1, qf[2 * j + 1], fmaf(k0, qf[2 * j], sacc));
      aacc = fmaf(fabsf(k1), fabsf(qf[2 * j + 1]), fmaf(fabsf(k0), fabsf(qf[2 * j]), aacc));
    }
    sv[u] = sacc;
    av[u] = aacc;
  }
  const bool b3 = hl & 8, b2 = hl & 4, b1 = hl & 2;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float ss = b3 ? sv[i] : sv[i + 4], sk = b3 ? sv[i + 4] : sv[i];
    const float as = b3 ? av[i] : av[i + 4], ak = b3 ? av[i + 4] : av[i];
    sv[i] = sk + __shfl_xor_sync(0xffffffffu, ss, 8);
    av[i] = ak + __shfl_xor_sync(0xffffffffu, as, 8);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float ss = b2 ? sv[i] : sv[i + 2], sk = b2 ? sv[i + 2] : sv[i];
    const float as = b2 ? av[i] : av[i + 2], ak = b2 ? av[i + 2] : av[i];
    sv[i] = sk + __shfl_xor_sync(0xffffffffu, ss, 4);
    av[i] = ak + __shfl_xor_sync(0xffffffffu, as, 4);
  }
  {
    const float ss = b1 ? sv[0] : sv[1], sk = b1 ? sv[1] : sv[0];
    const float as = b1 ? av[0] : av[1], ak = b1 ? av[1] : av[0];
    sv[0] = sk + __shfl_xor_sync(0xffffffffu, ss, 2);
    av[0] = ak + __shfl_xor_sync(0xffffffffu, as, 2);
  }
  sv[0] += __shfl_xor_sync(0xffffffffu, sv[0], 1);
  av[0] += __shfl_xor_sync(0xffffffffu, av[0], 1);
  const int u = (b3 ? 4 : 0) + (b2 ? 2 : 0) + (b1 ? 1 : 0);
  const int p = p0 + 2 * u + half;
  if (!(hl & 1) && p < pe) {
    const float s_ = sv[0], a_ = av[0];
    const float bound = (gam * a_ + kr * qmax) * 1.001f + fabsf(s_) * 2.4e-7f + 1e-30f;
    lo_out[p] = f2key(__fsub_rd(s_, bound));
    up_out[p] = __fadd_ru(s_, bound);
  }
}

// fp32 accumulation bound of the screen dot: (D+8) 2^-24 + 2^-23 (+ f64 slack)
__device__ __forceinline__ float screen_gamma(int D) { return (float)(D + 8) * 5.9604645e-08f + 1.1920929e-07f; }

__device__ __forceinline__ void screen_rows(const Dev& dv, int lbh, int pool_lo, int pb, int pe, const double* qsum,
                                            float qmax, unsigned* lo_out, float* up_out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int D = dv.D, E = D / 16, hl = lane & 15;
  const __nv_bfloat16* k16 = dv.kc16 + ((size_t)lbh * dv.NB + pool_lo) * D;
  const float* kerr = dv.kc_err + (size_t)lbh * dv.NB + pool_lo;
  float qf[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) qf[j] = j < E ? (float)qsum[hl * E + j] : 0.0f;
  for (int p0 = pb + warp * 16; p0 < pe; p0 += nwarps * 16) {
    uint4 raw[8];
    float kr;
    screen_load(k16, kerr, D, p0, pe, raw, kr);
    screen_finish(raw, qf, kr, screen_gamma(D), qmax, p0, pe, lo_out, up_out);
  }
}

template <bool SPLIT>
__device__ void screened_topk(const Dev& dv, int lbh, int pool_lo, int P, int m, SelSmem& sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int D = dv.D;
  if (SPLIT) {  // the intervals come from screen_scan_kernel (same stream, earlier)
    const unsigned* lo = dv.scr_lo + (size_t)lbh * dv.NB;
    const float* up = dv.scr_up + (size_t)lbh * dv.NB;
    for (int p = tid; p < P; p += blockDim.x) {
      sm.lo_key[p] = __ldcg(lo + p);
      sm.up[p] = __ldcg(up + p);
    }
  } else {
    screen_rows(dv, lbh, pool_lo, 0, P, sm.qsum, __int_as_float(sm.misc[M_QMAX]), sm.lo_key, sm.up);
  }
  __syncthreads();
  sel_mark(sm, 2);
  // (b) T = (a lower bound of) the m-th largest lower bound: two 8-bit radix passes fix the top
  //     16 bits of its key (sign, exponent, 7 mantissa bits: bins ~1% wide) and T is the bin's
  //     lower edge.  T at or below the exact m-th value keeps the candidate test exact; it only
  //     admits the few rows of the same bin.
  unsigned prefix = 0u, pmask = 0u;
  int remaining = m;
  for (int pass = 0; pass < 2; ++pass) {
    const int shift = 24 - 8 * pass;
    for (int i = tid; i < 256; i += blockDim.x) sm.hist[i] = 0;
    __syncthreads();
    for (int p = tid; p < P; p += blockDim.x) {
      const unsigned k = sm.lo_key[p];
      if ((k & pmask) == prefix) atomicAdd(&sm.hist[(k >> shift) & 255u], 1);
    }
    __syncthreads();
    if (warp == 0) {
      int c[8], sum = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        c[j] = sm.hist[255 - 8 * lane - j];
        sum += c[j];
      }
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      const int excl = incl - sum;
      if (excl < remaining && remaining <= incl) {
        int acc = excl;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (acc + c[j] >= remaining) {
            sm.misc[M_BIN] = 255 - 8 * lane - j;
            sm.misc[M_REM] = remaining - acc;
            break;
          }
          acc += c[j];
        }
      }
    }
    __syncthreads();
    prefix |= (unsigned)sm.misc[M_BIN] << shift;
    pmask |= 255u << shift;
    remaining = sm.misc[M_REM];
  }
  const float T = key2f(prefix);
  sel_mark(sm, 3);
  // (c) candidates: up >= T, rescored in f64 (one warp per row)
  if (tid == 0) sm.misc[M_NC] = 0;
  __syncthreads();
  for (int p = tid; p < P; p += blockDim.x)
    if (sm.up[p] >= T) sm.idx[atomicAdd(&sm.misc[M_NC], 1)] = p;
  __syncthreads();
  const int nc = sm.misc[M_NC];
  if (tid == 0) dv.stats[(size_t)lbh * ST_N + ST_CAND] += nc;
  double* cs = reinterpret_cast<double*>(sm.key);  // candidate scores
  const double* kc = dv.kc + ((size_t)lbh * dv.NB + pool_lo) * D;
  for (int i = warp; i < nc; i += 2 * nwarps) {  // two rows per warp in flight, same order as row_dot64
    const int i2 = i + nwarps;
    const double* r1 = kc + (size_t)sm.idx[i] * D;
    const double* r2 = kc + (size_t)sm.idx[i2 < nc ? i2 : i] * D;
    double a1 = 0.0, a2 = 0.0;
    for (int d = lane * 2; d < D; d += 64) {
      const double2 v1 = __ldg(reinterpret_cast<const double2*>(r1 + d));
      const double2 v2 = __ldg(reinterpret_cast<const double2*>(r2 + d));
      a1 = fma(v1.y, sm.qsum[d + 1], fma(v1.x, sm.qsum[d], a1));
      a2 = fma(v2.y, sm.qsum[d + 1], fma(v2.x, sm.qsum[d], a2));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      a1 += __shfl_xor_sync(0xffffffffu, a1, o);
      a2 += __shfl_xor_sync(0xffffffffu, a2, o);
    }
    if (lane == 0) {
      cs[i] = a1;
      if (i2 < nc) cs[i2] = a2;
    }
  }
  __syncthreads();
  sel_mark(sm, 4);
  // (d) rank the candidates by (score desc, index asc); the first m are the picks
  for (int i = tid; i < nc; i += blockDim.x) {
    const double si = cs[i];
    const int pi = sm.idx[i];
    int rank = 0;
    for (int j = 0; j < nc; ++j) {
      const double sj = cs[j];
      rank += (sj > si) || (sj == si && sm.idx[j] < pi);
    }
    if (rank < m) atomicOr(&sm.bm_q[pi >> 5], 1u << (pi & 31));
  }
  __syncthreads();
  sel_mark(sm, 5);
}

// ------------------------------------------------------------------------------------------
// Selection phase: fills sm.req[0..n_req) (sorted) and the selection buffers.
template <typename T, bool SPLIT>
__device__ void select_phase(const Dev& dv, int layer, int b, int h, const T* __restrict__ q,
                             int selector, SelSmem& sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int lbh = (layer * dv.B + b) * dv.H + h;
  const int D = dv.D, n_b = dv.n_b;
  const int t = dv.t[lbh], t0 = dv.t0[lbh];
  const int nblk = (t + n_b - 1) / n_b;                       // BlockGeometry.n_blocks
  const int recent_start = max(0, t0 - dv.n_w + 1);           // selection.py:49
  const int pool_lo = dv.n_sink;                              // selection.py:59
  const int pool_hi = max(pool_lo, recent_start / n_b);       // selection.py:60-61
  const int P = pool_hi - pool_lo;
  const int recent_lo = min(recent_start / n_b, nblk);        // selection.py:68-70
  const int a_end = min(dv.n_sink, nblk);                     // sink blocks < n_blocks(t)
  const int r_begin = max(recent_lo, a_end);
  const int Pp = next_pow2(P);

  // (1) q_sum = sum of the group's query heads (decode.py:171-172), f64 (split scan: the scan
  //     kernel computed and stored it)
  if (tid == 0) sm.misc[M_QMAX] = 0;
  __syncthreads();
  if (SPLIT) {
    for (int i = tid; i < D; i += blockDim.x) sm.qsum[i] = __ldcg(dv.qsum_buf + (size_t)lbh * D + i);
  } else for (int i = tid; i < D; i += blockDim.x) {
    const T* qg = q + ((size_t)b * dv.Hq + h * dv.G) * D + i;
    T v[8];
#pragma unroll
    for (int g = 0; g < 8; ++g) if (g < dv.G) v[g] = qg[(size_t)g * D];  // every load in flight
    double acc = 0.0;
#pragma unroll
    for (int g = 0; g < 8; ++g) if (g < dv.G) acc += to_f64(v[g]);        // in head order
    for (int g = 8; g < dv.G; ++g) acc += to_f64(qg[(size_t)g * D]);
    sm.qsum[i] = acc;
    if (dv.screen) {
      dv.qsum_buf[(size_t)lbh * D + i] = acc;
      const int bits = __float_as_int(__double2float_ru(fabs(acc)));  // |q| bits order as ints
      const int wmax = __reduce_max_sync(__activemask(), bits);
      if (lane == __ffs(__activemask()) - 1) atomicMax(&sm.misc[M_QMAX], wmax);
    }
  }
  __syncthreads();
  sel_mark(sm, 1);
  const int m_q_eff = min(selector == 0 ? dv.m_q : dv.m_topk, P);
  if (dv.screen) {
    for (int w = tid; w < Pp / 32; w += blockDim.x) {
      sm.bm_q[w] = 0u;
      sm.bm_e[w] = 0u;
    }
    __syncthreads();
    if (m_q_eff >= P) {  // the whole pool is picked: no scores needed
      for (int p = tid; p < P; p += blockDim.x) atomicOr(&sm.bm_q[p >> 5], 1u << (p & 31));
      __syncthreads();
    } else if (m_q_eff > 0) {
      screened_topk<SPLIT>(dv, lbh, pool_lo, P, m_q_eff, sm);
    }
  } else {

  // (2) s_q = K_c[pool] . q_sum.  Each warp streams 4 block rows per iteration; lane l holds
  //     dims [l*D/32, (l+1)*D/32) of every row, all loads issued before the FMAs, then a
  //     butterfly reduce-scatter leaves row (l>>3)&3 fully summed on lanes with l%8 == 0.
  //     (4 rows, not 8, keep the CTA within the 64-register budget of 4 CTAs per SM, so one
  //     CTA's scan overlaps another's sort and plan.)
  const double* kc = dv.kc + (size_t)lbh * dv.NB * D;
  double* s_q_out = dv.s_q + (size_t)lbh * dv.NB;
  const int nv = D / 64;  // double2 loads per lane per row (1 or 2)
  const double* qs = sm.qsum + lane * 2 * nv;
  for (int p0 = warp * 4; p0 < P; p0 += nwarps * 4) {
    double2 v[4][2];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int p = p0 + u;
      const double2* row = reinterpret_cast<const double2*>(kc + (size_t)(pool_lo + min(p, P - 1)) * D) + lane * nv;
      v[u][0] = __ldg(row);
      v[u][1] = nv == 2 ? __ldg(row + 1) : make_double2(0.0, 0.0);
    }
    double a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a[u] = fma(v[u][0].y, qs[1], v[u][0].x * qs[0]);
      if (nv == 2) a[u] = fma(v[u][1].y, qs[3], fma(v[u][1].x, qs[2], a[u]));
    }
    const bool b4 = lane & 16, b3 = lane & 8;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const double send = b4 ? a[i] : a[i + 2];
      const double keep = b4 ? a[i + 2] : a[i];
      a[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
    {
      const double send = b3 ? a[0] : a[1];
      const double keep = b3 ? a[1] : a[0];
      a[0] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    a[0] += __shfl_xor_sync(0xffffffffu, a[0], 4);
    a[0] += __shfl_xor_sync(0xffffffffu, a[0], 2);
    a[0] += __shfl_xor_sync(0xffffffffu, a[0], 1);
    const int p = p0 + (b4 ? 2 : 0) + (b3 ? 1 : 0);
    if ((lane & 7) == 0 && p < P) {
      sm.key[p] = order_key(a[0]);
      sm.idx[p] = p;
      s_q_out[pool_lo + p] = a[0];
    }
  }
  for (int p = P + tid; p < Pp; p += blockDim.x) {
    sm.key[p] = 0ull;
    sm.idx[p] = 0x7fffffff;
  }
  for (int w = tid; w < Pp / 32; w += blockDim.x) {
    sm.bm_q[w] = 0u;
    sm.bm_e[w] = 0u;
  }
  __syncthreads();

  // (3) query-aware top-k over the pool (argtopk order)
  if (P > 0) block_sort_best_first(sm.key, sm.idx, Pp);
  for (int r = tid; r < m_q_eff; r += blockDim.x) {
    const int p = sm.idx[r];
    atomicOr(&sm.bm_q[p >> 5], 1u << (p & 31));
  }
  __syncthreads();
  }  // full f64 scan

  // (4) NOSA: query-agnostic picks = first m_e pool blocks of the frozen s_e rank order that
  //     were not picked by the query (selection.py:151-156)
  if (selector == 0 && warp == 0) {
    const int m_e_eff = min(dv.m_e, P - m_q_eff);
    const int* rank = dv.rank_e + (size_t)lbh * dv.NB;
    // at most m_q_eff of the first m_q_eff + m_e_eff ranked blocks are query picks, so only
    // that prefix is read; 4 x 32 entries are loaded before any is used
    const int need = min(P, m_q_eff + m_e_eff);
    int cnt = 0;
    for (int g0 = 0; g0 < need && cnt < m_e_eff; g0 += 128) {
      int pr[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int i = g0 + 32 * k + lane;
        pr[k] = i < need ? __ldg(rank + i) : -1;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int p = pr[k];
        const bool ok = p >= 0 && !((sm.bm_q[p >> 5] >> (p & 31)) & 1u);
        const unsigned bal = __ballot_sync(0xffffffffu, ok);
        const int pos = cnt + __popc(bal & ((1u << lane) - 1u));
        if (ok && pos < m_e_eff) atomicOr(&sm.bm_e[p >> 5], 1u << (p & 31));
        cnt += __popc(bal);
      }
    }
  }
  __syncthreads();

  sel_mark(sm, 6);
  // (5) sorted outputs: blocks_q, blocks_e, required = sink U picked U recent, one part per warp
  const int nw = Pp / 32;
  int n_picked = 0;  // every thread counts the picks (broadcast reads of <= 32 words)
  for (int w = 0; w < nw; ++w) n_picked += __popc(sm.bm_q[w] | sm.bm_e[w]);
  const int n_req = a_end + n_picked + (nblk - r_begin);
  if (warp == 0) {
    const int nq = warp_bits_to_sorted(sm.bm_q, nw, pool_lo, dv.sel_q + (size_t)lbh * dv.MQ);
    if (lane == 0) {
      sm.misc[M_NQ] = nq;
      dv.n_selq[lbh] = nq;
      sm.misc[M_NREQ] = n_req;
    }
  } else if (warp == 1) {
    const int ne = warp_bits_to_sorted(sm.bm_e, nw, pool_lo, dv.sel_e + (size_t)lbh * dv.ME);
    if (lane == 0) {
      sm.misc[M_NE] = ne;
      dv.n_sele[lbh] = ne;
    }
  } else if (warp == 2) {  // merged picked list, after the sink part of req
    int n = 0;
    for (int w = 0; w < nw; ++w) {
      const unsigned word = sm.bm_q[w] | sm.bm_e[w];
      if (word == 0u) continue;
      if ((word >> lane) & 1u) {
        const int pos = a_end + n + __popc(word & ((1u << lane) - 1u));
        if (pos < dv.C) sm.req[pos] = pool_lo + w * 32 + lane;
      }
      n += __popc(word);
    }
  } else if (n_req <= dv.C) {  // sink and recent parts
    const int t3 = tid - 96, n3 = blockDim.x - 96;
    for (int j = t3; j < a_end; j += n3) sm.req[j] = j;
    for (int j = r_begin + t3; j < nblk; j += n3) sm.req[a_end + n_picked + (j - r_begin)] = j;
  }
  __syncthreads();
}

// ------------------------------------------------------------------------------------------
// Planning phase on sm.req[0..n_req): plan_transfers + apply_transfers for one manager.
__device__ void plan_phase(const Dev& dv, int layer, int b, int h, SelSmem& sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lbh = (layer * dv.B + b) * dv.H + h;
  const int C = dv.C, NB = dv.NB;
  int* slot_of = dv.slot_of + (size_t)lbh * NB;
  int* blk_of = dv.blk_of + (size_t)lbh * C;
  int* lastreq = dv.lastreq + (size_t)lbh * C;
  int* fstack = dv.fstack + (size_t)lbh * C;
  const int n_req = sm.misc[M_NREQ];

  if (n_req > C) {  // CapacityExceeded (kv_manager.py:215-219): no state change
    if (tid == 0) {
      atomicOr(dv.err, 1u);
      dv.n_req[lbh] = 0;
      dv.plan_n[lbh * 3 + 0] = 0;
      dv.plan_n[lbh * 3 + 1] = 0;
      dv.plan_n[lbh * 3 + 2] = 0;
    }
    return;
  }

  // (1) clock tick, hit test, fetch list in required order (kv_manager.py:212-229)
  if (warp == 0) {
    const int clock = dv.clock[lbh] + 1;
    int nf = 0;
    for (int g0 = 0; g0 < n_req; g0 += 128) {
      int blk[4], sl[4];  // 4 x 32 table lookups in flight before any is used
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int i = g0 + 32 * k + lane;
        blk[k] = i < n_req ? sm.req[i] : 0;
        sl[k] = i < n_req ? slot_of[blk[k]] : 0;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int i = g0 + 32 * k + lane;
        const bool miss = i < n_req && sl[k] < 0;
        if (i < n_req && sl[k] >= 0) {
          lastreq[sl[k]] = clock;
          sm.reqslot[i] = sl[k];
        }
        const unsigned bal = __ballot_sync(0xffffffffu, miss);
        if (miss) {
          const int pos = nf + __popc(bal & ((1u << lane) - 1u));
          sm.fetch[pos] = blk[k];
          sm.fpos[pos] = i;
        }
        nf += __popc(bal);
      }
    }
    if (lane == 0) {
      dv.clock[lbh] = clock;
      sm.misc[M_CLOCK] = clock;
      sm.misc[M_NF] = nf;
      sm.misc[M_SHORT] = nf - dv.ftop[lbh];  // shortfall (kv_manager.py:232)
      sm.misc[M_NCAND] = 0;
    }
  }
  __syncthreads();
  const int nf = sm.misc[M_NF];
  const int shortfall = sm.misc[M_SHORT];
  const int clock = sm.misc[M_CLOCK];

  sel_mark(sm, 8);
  // (2) victims: least-recently-required resident blocks not required now (kv_manager.py:233-246)
  if (shortfall > 0) {
    for (int s = tid; s < C; s += blockDim.x) {
      const int blk = blk_of[s];
      const bool cand = blk >= 0 && lastreq[s] != clock;
      sm.ckey[s] = cand ? ((unsigned long long)(unsigned)lastreq[s] << 32) | (unsigned)blk
                        : ~0ull;
      if (cand) atomicAdd(&sm.misc[M_NCAND], 1);
    }
    __syncthreads();
    for (int s = tid; s < C; s += blockDim.x) {
      const unsigned long long mine = sm.ckey[s];
      if (mine == ~0ull) continue;
      int rank = 0;
      for (int u = 0; u < C; ++u) rank += sm.ckey[u] < mine;
      if (rank < shortfall) sm.victims[rank] = s;
    }
    __syncthreads();
    if (sm.misc[M_NCAND] < shortfall) {  // cannot happen when n_req <= C; kept for parity
      if (tid == 0) atomicOr(dv.err, 1u);
      return;
    }
  }

  sel_mark(sm, 9);
  // (3) apply: evictions push their slots (LRR order), fetches pop (required order)
  if (warp == 0) {
    int top = dv.ftop[lbh];
    int* pe = dv.plan_evict + (size_t)lbh * C;
    int* pf = dv.plan_fetch + (size_t)lbh * C;
    const int nev = shortfall > 0 ? shortfall : 0;
    for (int r = lane; r < nev; r += 32) {
      const int s = sm.victims[r];
      const int blk = blk_of[s];
      slot_of[blk] = -1;
      blk_of[s] = -1;
      fstack[top + r] = s;
      pe[r] = blk;
    }
    __syncwarp();
    top += nev;
    const int t0 = dv.t0[lbh];
    int n_new = 0;
    for (int f = lane; f < nf; f += 32) {
      const int s = fstack[top - 1 - f];
      const int blk = sm.fetch[f];
      slot_of[blk] = s;
      blk_of[s] = blk;
      lastreq[s] = clock;
      sm.reqslot[sm.fpos[f]] = s;
      pf[f] = blk;
      n_new += (blk * dv.n_b >= t0);  // born during the run (offload_sim.py:286-289)
    }
    // top-k accounting: required blocks of the selection pool and the fetches among them
    const int rs_blk = max(0, t0 - dv.n_w + 1) / dv.n_b;
    int n_tk = 0, n_tkm = 0;
    for (int i = lane; i < n_req; i += 32) n_tk += sm.req[i] >= dv.n_sink && sm.req[i] < rs_blk;
    for (int f = lane; f < nf; f += 32) n_tkm += sm.fetch[f] >= dv.n_sink && sm.fetch[f] < rs_blk;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      n_new += __shfl_xor_sync(0xffffffffu, n_new, o);
      n_tk += __shfl_xor_sync(0xffffffffu, n_tk, o);
      n_tkm += __shfl_xor_sync(0xffffffffu, n_tkm, o);
    }
    top -= nf;
    // enqueue the misses for the gather (K3)
    int base = 0;
    if (lane == 0 && nf > 0) base = atomicAdd(dv.cnt + kCntStride * layer, nf);
    base = __shfl_sync(0xffffffffu, base, 0);
    int4* ml = dv.miss_list + (size_t)layer * dv.B * dv.H * C;
    // a block whose only token was appended at the previous step of this run is rebuilt from
    // the device-side stash of that row (the slow copy holds the same bytes)
    const int t_now = dv.t[lbh];
    // hybrid mover: this unit's misses go to the host-packed list (w = 2: the SM gather skips
    // them) or stay with the SM gather; a fixed hash of the unit splits the batch
    const bool to_host = dv.x_on && ((((unsigned)lbh * 2654435761u) >> 22) < (unsigned)dv.x_split);
    for (int f = lane; f < nf; f += 32) {
      const int blk = sm.fetch[f];
      const int born = (blk * dv.n_b == t_now - 1) && (t_now - 1 >= t0);
      ml[base + f] = make_int4(lbh, blk, sm.reqslot[sm.fpos[f]], born ? 1 : (to_host ? 2 : 0));
    }
    if (to_host) {
      // copy list for the host: every miss but a block born by the last append (rebuilt on the
      // device; it is the newest block, so always the last fetch); the layer's last CTA then
      // publishes the counts (select_plan_kernel)
      const int last_born = nf > 0 && sm.fetch[nf - 1] * dv.n_b == t_now - 1 && t_now - 1 >= t0;
      const int nx = nf - last_born;
      int xb = 0;
      if (lane == 0 && nx > 0) xb = atomicAdd(dv.cnt + kCntStride * layer + 2, nx);
      xb = __shfl_sync(0xffffffffu, xb, 0);
      const size_t cap = (size_t)dv.B * dv.H * C;
      for (int f = lane; f < nx; f += 32) {
        const int blk = sm.fetch[f];
        dv.x_src[layer * cap + xb + f] = const_cast<char*>(dv.x_src_base) + ((size_t)lbh * dv.NB + blk) * dv.bpb;
        dv.x_dst[layer * cap + xb + f] = dv.pool + ((size_t)lbh * C + sm.reqslot[sm.fpos[f]]) * dv.bpb;
      }
    }
    if (lane == 0) {
      dv.ftop[lbh] = top;
      long long* st = dv.stats + (size_t)lbh * ST_N;
      st[ST_HITS] += n_req - nf;
      st[ST_MISSES] += nf;
      st[ST_NEW] += n_new;
      st[ST_EVICT] += nev;
      st[ST_STEPS] += 1;
      st[ST_TOPK] += n_tk;
      st[ST_TOPK_MISS] += n_tkm;
      dv.plan_n[lbh * 3 + 0] = nf;
      dv.plan_n[lbh * 3 + 1] = nev;
      dv.plan_n[lbh * 3 + 2] = n_req - nf;
      dv.n_req[lbh] = n_req;
    }
  }
  __syncthreads();
  for (int i = tid; i < n_req; i += blockDim.x) {
    dv.req[(size_t)lbh * C + i] = sm.req[i];
    dv.req_slot[(size_t)lbh * C + i] = sm.reqslot[i];
  }
  if (dv.born_local && nf > 0) {
    // all-resident run: the misses are blocks born by the last append (still counted as misses,
    // offload_sim.py:286-289); the planner writes them into their new slots itself, so the
    // step launches no gather.  Any other miss would break that invariant: flagged.
    const int t_now = dv.t[lbh], t0 = dv.t0[lbh];
    for (int f = 0; f < nf; ++f) {
      const int blk = sm.fetch[f];
      if (blk * dv.n_b == t_now - 1 && t_now - 1 >= t0) {
        const int s = sm.reqslot[sm.fpos[f]];
        write_born_block(dv, make_int4(lbh, blk, s, 1), reinterpret_cast<int4*>(dv.pool + ((size_t)lbh * C + s) * dv.bpb),
                         (int)(dv.bpb / 16));
      } else if (tid == 0) {
        atomicOr(dv.err, 4u);
      }
    }
  }
}

// Screen scan as its own kernel (Dev::split_scan): grid = (row chunks, B*H, layers), 256 threads.
// Every CTA sums its unit's query group (the same f64 order as select_phase) and screens its
// chunk of pool rows (`rows`, a multiple of 128; by default the whole pool) into the global
// interval scratch, 128 rows per iteration with the next iteration's rows already in flight;
// chunk 0 also stores q_sum for the f64 rescoring.  Purely bandwidth-bound (the bf16 K_c rows
// are the bytes), so it streams at full occupancy instead of alternating with the selection's
// latency-bound phases.
template <typename T>
__global__ void __launch_bounds__(256) screen_scan_kernel(Dev dv, int layer0, const T* __restrict__ q0,
                                                          size_t q_layer_stride, int rows) {
  __shared__ float qt[128];  // (float) q_sum, transposed [j][hl]: conflict-free qf loads
  __shared__ int qmax_bits;
  const int layer = layer0 + blockIdx.z;
  const T* q = q0 + blockIdx.z * q_layer_stride;
  const int bh = blockIdx.y, b = bh / dv.H, h = bh % dv.H;
  const int lbh = (layer * dv.B + b) * dv.H + h;
  const int D = dv.D, E = D / 16, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int t0 = dv.t0[lbh];
  const int recent_start = max(0, t0 - dv.n_w + 1);           // selection.py:49
  const int pool_lo = dv.n_sink;                              // selection.py:59
  const int P = max(pool_lo, recent_start / dv.n_b) - pool_lo;
  const int pb = blockIdx.x * rows, pe = min(pb + rows, P);
  if (pb >= max(P, 1)) return;  // (chunk 0 always runs: it stores q_sum)
  // the pool rows do not depend on q: their loads are in flight while q_sum is formed
  const __nv_bfloat16* k16 = dv.kc16 + ((size_t)lbh * dv.NB + pool_lo) * D;
  const float* kerr = dv.kc_err + (size_t)lbh * dv.NB + pool_lo;
  const int stride = nwarps * 16;
  int p0 = pb + warp * 16;
  uint4 raw[8];
  float kr = 0.0f;
  if (p0 < pe) screen_load(k16, kerr, D, p0, pe, raw, kr);
  if (tid == 0) qmax_bits = 0;
  __syncthreads();
  for (int i = tid; i < D; i += blockDim.x) {
    const T* qg = q + ((size_t)b * dv.Hq + h * dv.G) * D + i;
    T v[8];
#pragma unroll
    for (int g = 0; g < 8; ++g) if (g < dv.G) v[g] = qg[(size_t)g * D];
    double acc = 0.0;
#pragma unroll
    for (int g = 0; g < 8; ++g) if (g < dv.G) acc += to_f64(v[g]);  // the order of select_phase
    for (int g = 8; g < dv.G; ++g) acc += to_f64(qg[(size_t)g * D]);
    qt[(i % E) * 16 + i / E] = (float)acc;
    const int bits = __float_as_int(__double2float_ru(fabs(acc)));  // |q| bits order as ints
    const int wmax = __reduce_max_sync(__activemask(), bits);
    if ((tid & 31) == __ffs(__activemask()) - 1) atomicMax(&qmax_bits, wmax);
    if (blockIdx.x == 0) dv.qsum_buf[(size_t)lbh * D + i] = acc;
  }
  __syncthreads();
  if (p0 >= pe) return;
  const int hl = lane & 15;
  float qf[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) qf[j] = j < E ? qt[j * 16 + hl] : 0.0f;
  unsigned* lo = dv.scr_lo + (size_t)lbh * dv.NB;
  float* up = dv.scr_up + (size_t)lbh * dv.NB;
  const float qmax = __int_as_float(qmax_bits), gam = screen_gamma(D);
  for (;;) {
    const int p1 = p0 + stride;
    uint4 nxt[8];
    float kn = 0.0f;
    if (p1 < pe) screen_load(k16, kerr, D, p1, pe, nxt, kn);  // next iteration's rows in flight
    screen_finish(raw, qf, kr, gam, qmax, p0, pe, lo, up);
    if (p1 >= pe) break;
#pragma unroll
    for (int u = 0; u < 8; ++u) raw[u] = nxt[u];
    kr = kn;
    p0 = p1;
  }
}

// grid = (B*H, layers), block = 256: layer = layer0 + blockIdx.y with its queries at
// q + blockIdx.y * q_layer_stride.  mode: 0 = select only, 1 = select + plan, 2 = plan on ext_req.
// SPLIT: the screen scan ran as screen_scan_kernel (no scan code here: fewer registers, more CTAs
// per SM); otherwise 4 CTAs per SM so that one CTA's scan overlaps another's sort/plan.
#ifndef SEL_SPLIT_CTAS
#define SEL_SPLIT_CTAS 5
#endif
template <typename T, bool SPLIT>
__global__ void __launch_bounds__(256, SPLIT ? SEL_SPLIT_CTAS : 4)
    select_plan_kernel(Dev dv, int layer0, const T* __restrict__ q0, size_t q_layer_stride, int selector,
                       int mode, const int* __restrict__ ext_req, const int* __restrict__ ext_nreq) {
  extern __shared__ __align__(16) char smem_raw[];
  const int layer = layer0 + blockIdx.y;
  const T* q = q0 + blockIdx.y * q_layer_stride;
  const int bh = blockIdx.x;
  const int b = bh / dv.H, h = bh % dv.H;
  const int lbh = (layer * dv.B + b) * dv.H + h;
  const int Pp = next_pow2(dv.NB);
  SelSmem sm = carve_sel_smem(smem_raw, dv.D, Pp, dv.C);
  __shared__ long long marks[16];
  sm.marks = dv.sel_prof ? marks : nullptr;
  if (sm.marks && threadIdx.x == 0)
    for (int i = 0; i < 16; ++i) marks[i] = 0;
  sel_mark(sm, 0);

  if (mode == 2) {
    const int n = ext_nreq[bh];
    if (n < 0) return;  // this manager is not part of the call: no clock tick, no stats
    if (threadIdx.x == 0) sm.misc[M_NREQ] = n;
    for (int i = threadIdx.x; i < min(n, dv.C); i += blockDim.x) sm.req[i] = ext_req[(size_t)bh * dv.C + i];
    __syncthreads();
  } else {
    select_phase<T, SPLIT>(dv, layer, b, h, q, selector, sm);
  }
  if (mode == 0) {
    if (threadIdx.x == 0) dv.n_req[lbh] = min(sm.misc[M_NREQ], dv.C);
    for (int i = threadIdx.x; i < min(sm.misc[M_NREQ], dv.C); i += blockDim.x)
      dv.req[(size_t)lbh * dv.C + i] = sm.req[i];
    return;
  }
  sel_mark(sm, 7);
  plan_phase(dv, layer, b, h, sm);
  __syncthreads();
  if (dv.x_on && threadIdx.x == 0) {
    // the layer's last CTA publishes the exported miss counts to the host (every CTA gets here,
    // CapacityExceeded included); kernel completion makes them visible to the host
    __threadfence();
    if (atomicAdd(dv.cnt + kCntStride * layer + 3, 1) == (int)gridDim.x - 1) {
      __threadfence();
      const int total = atomicAdd(dv.cnt + kCntStride * layer, 0);
      const int xn = atomicAdd(dv.cnt + kCntStride * layer + 2, 0);
      reinterpret_cast<volatile int*>(dv.x_cnt)[2 * layer] = xn;
      reinterpret_cast<volatile int*>(dv.x_cnt)[2 * layer + 1] = total - xn;
    }
  }
  sel_mark(sm, 11);
  if (sm.marks && threadIdx.x == 0) {  // cycles per phase, summed over CTAs; [15] counts CTAs
    long long prev = marks[0];
    for (int i = 1; i < 12; ++i) {
      if (marks[i] == 0) continue;  // phase skipped
      atomicAdd(reinterpret_cast<unsigned long long*>(dv.sel_prof + i), (unsigned long long)(marks[i] - prev));
      prev = marks[i];
    }
    atomicAdd(reinterpret_cast<unsigned long long*>(dv.sel_prof + 15), 1ull);
  }
}

// ------------------------------------------------------------------------------------------
// start_run: freeze the geometry at the current length and rank the frozen pool by the
// query-agnostic block score (score desc, index asc).  grid = (#lbh in range), block = 256.
__global__ void __launch_bounds__(256) start_run_kernel(Dev dv, int seq_begin, int seq_count) {
  extern __shared__ __align__(16) char smem_raw[];
  const int i = blockIdx.x;  // over layers x seq_count x H
  const int h = i % dv.H;
  const int s = (i / dv.H) % seq_count;
  const int l = i / (dv.H * seq_count);
  const int lbh = (l * dv.B + seq_begin + s) * dv.H + h;
  const int t = dv.t[lbh];
  const int recent_start = max(0, t - dv.n_w + 1);
  const int pool_lo = dv.n_sink;
  const int pool_hi = max(pool_lo, recent_start / dv.n_b);
  const int P = pool_hi - pool_lo;
  const int Pp = next_pow2(P);
  unsigned long long* key = reinterpret_cast<unsigned long long*>(smem_raw);
  int* idx = reinterpret_cast<int*>(key + Pp);
  const double* se = dv.se + (size_t)lbh * dv.NB;
  for (int p = threadIdx.x; p < Pp; p += blockDim.x) {
    key[p] = p < P ? order_key(se[pool_lo + p]) : 0ull;
    idx[p] = p < P ? p : 0x7fffffff;
  }
  __syncthreads();
  if (P > 0) block_sort_best_first(key, idx, Pp);
  int* rank = dv.rank_e + (size_t)lbh * dv.NB;
  for (int p = threadIdx.x; p < P; p += blockDim.x) rank[p] = idx[p];
  if (threadIdx.x == 0) dv.t0[lbh] = t;
}

// ------------------------------------------------------------------------------------------
// Screened-selection state of the frozen pool, built at start_run: bf16(K_c) of every pool
// row and the L1 norm of its rounding error (rounded up).  One warp per row.
__global__ void __launch_bounds__(256) screen_build_kernel(Dev dv, int seq_begin, int seq_count) {
  const int i = blockIdx.x;  // over layers x seq_count x H
  const int h = i % dv.H;
  const int s = (i / dv.H) % seq_count;
  const int l = i / (dv.H * seq_count);
  const int lbh = (l * dv.B + seq_begin + s) * dv.H + h;
  const int D = dv.D, lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int recent_start = max(0, dv.t0[lbh] - dv.n_w + 1);
  const int pool_lo = dv.n_sink, pool_hi = max(pool_lo, recent_start / dv.n_b);
  for (int p = pool_lo + warp; p < pool_hi; p += nwarps) {
    const double* row = dv.kc + ((size_t)lbh * dv.NB + p) * D;
    __nv_bfloat16* out = dv.kc16 + ((size_t)lbh * dv.NB + p) * D;
    double e = 0.0;
    for (int d = lane; d < D; d += 32) {
      const double x = row[d];
      const __nv_bfloat16 y = __double2bfloat16(x);
      out[d] = y;
      e += fabs(x - (double)__bfloat162float(y));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
    if (lane == 0) dv.kc_err[(size_t)lbh * dv.NB + p] = __double2float_ru(e * (1.0 + 1e-12));
  }
}

// Parity readback of the screened selector: s_q of every pool row in f64, from the step's q_sum,
// in the refinement's order (row_dot64).  grid = B*H of one layer.
__global__ void __launch_bounds__(256) score_readback_kernel(Dev dv, int layer) {
  const int lbh = layer * dv.B * dv.H + blockIdx.x;
  const int D = dv.D, lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int recent_start = max(0, dv.t0[lbh] - dv.n_w + 1);
  const int pool_lo = dv.n_sink, pool_hi = max(pool_lo, recent_start / dv.n_b);
  extern __shared__ double qsum_sm[];
  for (int i = threadIdx.x; i < D; i += blockDim.x) qsum_sm[i] = dv.qsum_buf[(size_t)lbh * D + i];
  __syncthreads();
  for (int p = pool_lo + warp; p < pool_hi; p += nwarps) {
    const double v = row_dot64(dv.kc + ((size_t)lbh * dv.NB + p) * D, qsum_sm, D);
    if (lane == 0) dv.s_q[(size_t)lbh * dv.NB + p] = v;
  }
}

cudaError_t launch_screen_build(const Dev& dv, int seq_begin, int seq_count, cudaStream_t st) {
  screen_build_kernel<<<dv.L * seq_count * dv.H, 256, 0, st>>>(dv, seq_begin, seq_count);
  return cudaGetLastError();
}

cudaError_t launch_score_readback(const Dev& dv, int layer, cudaStream_t st) {
  score_readback_kernel<<<dv.B * dv.H, 256, dv.D * sizeof(double), st>>>(dv, layer);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// Standalone selector on caller-provided block scores (nosa_select / infllmv2_select).
__global__ void __launch_bounds__(256)
    select_scores_kernel(const double* __restrict__ s_q, const double* __restrict__ s_e,
                         int stride, const int* __restrict__ pool_lo_a,
                         const int* __restrict__ pool_hi_a, int m_q, int m_e, int selector,
                         int* out_q, int* n_q, int* out_e, int* n_e, int Pp) {
  extern __shared__ __align__(16) char smem_raw[];
  unsigned long long* key = reinterpret_cast<unsigned long long*>(smem_raw);
  int* idx = reinterpret_cast<int*>(key + Pp);
  unsigned* bm_q = reinterpret_cast<unsigned*>(idx + Pp);
  unsigned* bm_e = bm_q + Pp / 32;
  const int prob = blockIdx.x;
  const int lo = pool_lo_a[prob];
  const int P = max(0, pool_hi_a[prob] - lo);
  const int Ps = next_pow2(P);
  const double* sq = s_q + (size_t)prob * stride;
  for (int p = threadIdx.x; p < Ps; p += blockDim.x) {
    key[p] = p < P ? order_key(sq[lo + p]) : 0ull;
    idx[p] = p < P ? p : 0x7fffffff;
  }
  for (int w = threadIdx.x; w < Ps / 32; w += blockDim.x) bm_q[w] = bm_e[w] = 0u;
  __syncthreads();
  if (P > 0) block_sort_best_first(key, idx, Ps);
  const int mq = min(m_q, P);
  for (int r = threadIdx.x; r < mq; r += blockDim.x) atomicOr(&bm_q[idx[r] >> 5], 1u << (idx[r] & 31));
  __syncthreads();
  if (selector == 0) {
    // second phase over the rest: picked_q keys sink below every real score
    const double* se = s_e + (size_t)prob * stride;
    for (int p = threadIdx.x; p < Ps; p += blockDim.x) {
      const bool picked = p < P && ((bm_q[p >> 5] >> (p & 31)) & 1u);
      key[p] = (p < P && !picked) ? order_key(se[lo + p]) : 0ull;
      idx[p] = (p < P && !picked) ? p : 0x7fffffff;
    }
    __syncthreads();
    if (P > 0) block_sort_best_first(key, idx, Ps);
    const int me = min(m_e, P - mq);
    for (int r = threadIdx.x; r < me; r += blockDim.x) atomicOr(&bm_e[idx[r] >> 5], 1u << (idx[r] & 31));
    __syncthreads();
  }
  if ((threadIdx.x >> 5) == 0) {
    const int cq = warp_bits_to_sorted(bm_q, Ps / 32, lo, out_q + (size_t)prob * max(m_q, 1));
    const int ce = warp_bits_to_sorted(bm_e, Ps / 32, lo, out_e + (size_t)prob * max(m_e, 1));
    if ((threadIdx.x & 31) == 0) {
      n_q[prob] = cq;
      n_e[prob] = ce;
    }
  }
}

// ------------------------------------------------------------------------------------------
// Shared-pool planner: the reference simulator's residency (offload_sim.py:254-299) — one fast
// pool of B*C slots per (layer, head) shared by every sequence, plan + apply per sequence in
// batch order, least-recently-required victims over all sequences by (clock, batch, block)
// (kv_manager.py:125-127), LIFO slot reuse.  Inherently serial in b: one CTA per head.
constexpr int kSharedThreads = 512;

__global__ void __launch_bounds__(kSharedThreads)
    plan_shared_kernel(Dev dv, int layer, const int* __restrict__ ext_req, const int* __restrict__ ext_nreq) {
  extern __shared__ __align__(16) char smem_raw[];
  const int h = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int B = dv.B, C = dv.C, H = dv.H, NB = dv.NB, N = B * C;
  int* req = reinterpret_cast<int*>(smem_raw);      // [C]
  int* reqslot = req + C;                           // [C] shared slot ids
  int* fetch = reqslot + C;                         // [C]
  int* fpos = fetch + C;                            // [C]
  int* victims = fpos + C;                          // [C]
  unsigned* chosen = reinterpret_cast<unsigned*>(victims + C);  // [N/32 + 1] bitmap
  unsigned long long* red_k = reinterpret_cast<unsigned long long*>(chosen + N / 32 + 2);  // [32]
  int* red_s = reinterpret_cast<int*>(red_k + 32);  // [32]
  int* misc = red_s + 32;                           // [8]
  const size_t head0 = (size_t)(layer * B) * H + h;  // (layer, b = 0, h): per-(layer, head) scalars
  if (tid == 0) {
    misc[0] = dv.clock[head0];
    misc[1] = dv.ftop[head0];
  }
  __syncthreads();
  for (int b = 0; b < B; ++b) {
    const int lbh = (layer * B + b) * H + h;
    const int n = ext_nreq ? ext_nreq[b * H + h] : dv.n_req[lbh];
    if (n < 0) continue;  // not part of this call
    if (n > C) {          // CapacityExceeded for this sequence's share (kv_manager.py:215-219)
      if (tid == 0) {
        atomicOr(dv.err, 1u);
        dv.n_req[lbh] = 0;
      }
      continue;
    }
    for (int i = tid; i < n; i += blockDim.x) req[i] = ext_req ? ext_req[((size_t)b * H + h) * C + i] : dv.req[(size_t)lbh * C + i];
    for (int w = tid; w < N / 32 + 1; w += blockDim.x) chosen[w] = 0u;
    __syncthreads();
    const int clock = misc[0] + 1;
    // (1) hit test and fetch list in required order
    if (warp == 0) {
      int nf = 0;
      for (int base = 0; base < n; base += 32) {
        const int i = base + lane;
        const int blk = i < n ? req[i] : 0;
        const int s = i < n ? dv.slot_of[(size_t)lbh * NB + blk] : 0;
        const bool miss = i < n && s < 0;
        if (i < n && s >= 0) {
          dv.lastreq[shared_idx(dv, layer, h, s)] = clock;
          reqslot[i] = s;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, miss);
        if (miss) {
          const int pos = nf + __popc(bal & ((1u << lane) - 1u));
          fetch[pos] = blk;
          fpos[pos] = i;
        }
        nf += __popc(bal);
      }
      if (lane == 0) {
        misc[0] = clock;
        misc[2] = nf;
        misc[3] = nf - misc[1];  // shortfall against the shared free list
      }
    }
    __syncthreads();
    const int nf = misc[2], shortfall = misc[3];
    // (2) victims: repeated block-wide argmin of (last_required, batch, block) over the pool,
    //     excluding blocks required now (they carry this call's clock)
    for (int r = 0; r < shortfall; ++r) {
      unsigned long long best = ~0ull;
      int best_s = -1;
      for (int s = tid; s < N; s += blockDim.x) {
        const size_t x = shared_idx(dv, layer, h, s);
        const int key = dv.blk_of[x];
        if (key < 0 || dv.lastreq[x] == clock || ((chosen[s >> 5] >> (s & 31)) & 1u)) continue;
        const unsigned long long k = ((unsigned long long)(unsigned)dv.lastreq[x] << 32) |
                                     ((unsigned long long)(key / NB) << 16) | (unsigned long long)(key % NB);
        if (k < best) { best = k; best_s = s; }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const unsigned long long ok = __shfl_xor_sync(0xffffffffu, best, o);
        const int os = __shfl_xor_sync(0xffffffffu, best_s, o);
        if (ok < best) { best = ok; best_s = os; }
      }
      if (lane == 0) { red_k[warp] = best; red_s[warp] = best_s; }
      __syncthreads();
      if (tid == 0) {
        unsigned long long k = ~0ull;
        int s = -1;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
          if (red_k[w] < k) { k = red_k[w]; s = red_s[w]; }
        victims[r] = s;
        if (s >= 0) chosen[s >> 5] |= 1u << (s & 31);
        else atomicOr(dv.err, 1u);  // not enough evictable blocks
      }
      __syncthreads();
    }
    // (3) apply: victims release their slots in LRR order, fetches pop in required order
    if (tid == 0) {
      int top = misc[1];
      const int nev = shortfall > 0 ? shortfall : 0;
      int* pe = dv.plan_evict + (size_t)lbh * C;
      int* pf = dv.plan_fetch + (size_t)lbh * C;
      for (int r = 0; r < nev; ++r) {
        const int s = victims[r];
        if (s < 0) break;
        const size_t x = shared_idx(dv, layer, h, s);
        const int key = dv.blk_of[x];
        dv.slot_of[(size_t)((layer * B + key / NB) * H + h) * NB + key % NB] = -1;
        dv.blk_of[x] = -1;
        dv.fstack[shared_idx(dv, layer, h, top + r)] = s;
        pe[r] = key;  // owner * NB + block
      }
      top += nev;
      const int t = dv.t[lbh], t0 = dv.t0[lbh];
      int n_new = 0;
      int base = nf ? atomicAdd(dv.cnt + kCntStride * layer, nf) : 0;
      int4* ml = dv.miss_list + (size_t)layer * B * H * C;
      for (int f = 0; f < nf; ++f) {
        const int s = dv.fstack[shared_idx(dv, layer, h, top - 1 - f)];
        const int blk = fetch[f];
        const size_t x = shared_idx(dv, layer, h, s);
        dv.slot_of[(size_t)lbh * NB + blk] = s;
        dv.blk_of[x] = b * NB + blk;
        dv.lastreq[x] = clock;
        reqslot[fpos[f]] = s;
        pf[f] = blk;
        n_new += blk * dv.n_b >= t0;
        const int born = (blk * dv.n_b == t - 1) && (t - 1 >= t0);
        ml[base + f] = make_int4(lbh, blk, shared_rel(dv, b, s), born);
      }
      top -= nf;
      misc[1] = top;
      const int rs_blk = max(0, t0 - dv.n_w + 1) / dv.n_b;
      int n_tk = 0, n_tkm = 0;
      for (int i = 0; i < n; ++i) n_tk += req[i] >= dv.n_sink && req[i] < rs_blk;
      for (int f = 0; f < nf; ++f) n_tkm += fetch[f] >= dv.n_sink && fetch[f] < rs_blk;
      long long* st = dv.stats + (size_t)lbh * ST_N;
      st[ST_TOPK] += n_tk;
      st[ST_TOPK_MISS] += n_tkm;
      st[ST_HITS] += n - nf;
      st[ST_MISSES] += nf;
      st[ST_NEW] += n_new;
      st[ST_EVICT] += nev;
      st[ST_STEPS] += 1;
      dv.plan_n[lbh * 3 + 0] = nf;
      dv.plan_n[lbh * 3 + 1] = nev;
      dv.plan_n[lbh * 3 + 2] = n - nf;
      dv.n_req[lbh] = n;
    }
    __syncthreads();
    for (int i = tid; i < n; i += blockDim.x) {
      dv.req[(size_t)lbh * C + i] = req[i];
      dv.req_slot[(size_t)lbh * C + i] = shared_rel(dv, b, reqslot[i]);
    }
    __syncthreads();
  }
  if (tid == 0) {
    dv.clock[head0] = misc[0];
    dv.ftop[head0] = misc[1];
  }
}

cudaError_t launch_plan_shared(const Dev& dv, int layer, const int* ext_req, const int* ext_nreq, cudaStream_t st) {
  const int N = dv.B * dv.C;
  const size_t smem = 5 * (size_t)dv.C * 4 + ((size_t)N / 32 + 2) * 4 + 32 * 8 + 32 * 4 + 8 * 4 + 64;
  cudaFuncSetAttribute(plan_shared_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  max_shared_carveout(plan_shared_kernel);
  plan_shared_kernel<<<dv.H, kSharedThreads, smem, st>>>(dv, layer, ext_req, ext_nreq);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// host-side launchers
cudaError_t launch_select_plan(const Dev& dv, int layer, const void* q, int selector, int mode,
                               const int* ext_req, const int* ext_nreq, cudaStream_t st, int layers) {
  int Pp = 32;
  while (Pp < dv.NB) Pp <<= 1;
  const size_t smem = sel_smem_bytes(dv.D, Pp, dv.C);
  const size_t qs = (size_t)dv.B * dv.Hq * dv.D;  // elements per layer of q
  const dim3 grid(dv.B * dv.H, layers);
  const bool split = dv.screen && dv.split_scan;  // (mode 2 plans only: the selection code never runs)
  if (mode != 2 && split) {
    // rows per CTA: the whole pool (one CTA per unit, the rows of the next 128-row iteration in
    // flight); NOSA_SCAN_ROWS=128 gives one 128-row chunk per CTA (the first split kernel)
    static const int env_rows = getenv("NOSA_SCAN_ROWS") ? std::max(1, atoi(getenv("NOSA_SCAN_ROWS"))) : 0;
    const int rows = env_rows ? (env_rows + 127) / 128 * 128 : (dv.NB + 127) / 128 * 128;
    const dim3 sgrid((dv.NB + rows - 1) / rows, dv.B * dv.H, layers);
    if (dv.dtype == 0)
      screen_scan_kernel<__nv_bfloat16><<<sgrid, 256, 0, st>>>(dv, layer, static_cast<const __nv_bfloat16*>(q), qs, rows);
    else
      screen_scan_kernel<float><<<sgrid, 256, 0, st>>>(dv, layer, static_cast<const float*>(q), qs, rows);
  }
  if (dv.dtype == 0) {
    auto k = split ? select_plan_kernel<__nv_bfloat16, true> : select_plan_kernel<__nv_bfloat16, false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    max_shared_carveout(k);
    k<<<grid, 256, smem, st>>>(dv, layer, static_cast<const __nv_bfloat16*>(q), qs, selector, mode, ext_req,
                               ext_nreq);
  } else {
    auto k = split ? select_plan_kernel<float, true> : select_plan_kernel<float, false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    max_shared_carveout(k);
    k<<<grid, 256, smem, st>>>(dv, layer, static_cast<const float*>(q), qs, selector, mode, ext_req, ext_nreq);
  }
  return cudaGetLastError();
}

cudaError_t launch_start_run(const Dev& dv, int seq_begin, int seq_count, cudaStream_t st) {
  int Pp = 32;
  while (Pp < dv.NB) Pp <<= 1;
  const size_t smem = (size_t)Pp * 12;
  cudaFuncSetAttribute(start_run_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  start_run_kernel<<<dv.L * seq_count * dv.H, 256, smem, st>>>(dv, seq_begin, seq_count);
  return cudaGetLastError();
}

cudaError_t launch_select_scores(int n_prob, const double* s_q, const double* s_e, int stride,
                                 const int* lo, const int* hi, int m_q, int m_e, int selector,
                                 int* out_q, int* n_q, int* out_e, int* n_e, cudaStream_t st) {
  int Pp = 32;
  while (Pp < stride) Pp <<= 1;
  const size_t smem = (size_t)Pp * 12 + 2 * (size_t)(Pp / 32) * 4;
  cudaFuncSetAttribute(select_scores_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  select_scores_kernel<<<n_prob, 256, smem, st>>>(s_q, s_e, stride, lo, hi, m_q, m_e, selector,
                                                  out_q, n_q, out_e, n_e, Pp);
  return cudaGetLastError();
}

}  // namespace nosa
