// nosa_project.cu — the QKV projection in front of the decode step (SURVEY.md §8f row 1:
// project_qkv, attention.py:67-90; DecodeEngine.step decode.py:162-164) as a tcgen05 GEMM.
//
//   C[M][N] = A[M][K] · B[N][K]ᵀ,  A = hidden states (bf16, row-major), B = the concatenated
//   [W_q | W_k | W_v] transposed to [N][K] (bf16, K-major), fp32 accumulation in TMEM.
//
// Grid (N/256, ceil(M/128), splits), clusters of `splits` CTAs along K.  Each CTA:
//   warp 0 lane 0  TMA producer: 64-wide bf16 boxes (128B swizzle), up to 128 rows of A and PN
//                  of B per stage, into a 6-stage ring (4 at PN = 256), one mbarrier per stage;
//   warp 1 lane 0  MMA issuer: tcgen05.mma M=128 N=256 K=16 (4 per stage) into a 256-column
//                  TMEM accumulator, tcgen05.commit frees each stage;
//   all 4 warps    epilogue: tcgen05.ld of the accumulator (warp w = TMEM lanes 32w..).
// One split: each thread converts its row to bf16 and stores it straight into q | k | v.
// Split-K: the partial tiles go to each CTA's shared memory and are summed across the cluster
// through distributed shared memory in rank order (deterministic, no global workspace, no
// second launch): CTA rank j reduces rows [j*128/S, (j+1)*128/S) of the tile and writes them.
// The A boxes hold the m-tile's rows only (M rounded up to 8 for decode-sized m).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "nosa_device.cuh"

namespace nosa {

constexpr int PM = 128, PK = 64, PTHREADS = 128;
constexpr int P_A_BYTES = PM * PK * 2;  // 16 KiB A box per stage
constexpr int P_MAX_SPLITS = 8;            // portable cluster size

// UMMA shared-memory descriptor: K-major operand, 128B swizzle, 8-row atoms 1024 B apart
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);  // start address (16 B units)        [0,14)
  d |= (uint64_t)1 << 16;                    // leading byte offset (unused: SW128 K-major)
  d |= (uint64_t)(1024 >> 4) << 32;          // stride byte offset: next 8-row group [32,46)
  d |= (uint64_t)1 << 46;                    // descriptor version (sm100)          [46,48)
  d |= (uint64_t)2 << 61;                    // layout: SWIZZLE_128B                [61,64)
  return d;
}

// instruction descriptor of kind::f16: bf16 x bf16 -> f32, both operands K-major
__host__ __device__ constexpr uint32_t idesc_bf16_f32(int m, int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

// 3-D box load: coordinates (k, row, layer)
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// (not volatile: the loads of all ranks may be issued back to back; the cluster barriers order
// them against the partial-tile writes)
__device__ __forceinline__ float4 ld_dsmem_f4(uint32_t local_addr, uint32_t rank) {
  uint32_t raddr;
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(local_addr), "r"(rank));
  float4 v;
  asm("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(raddr));
  return v;
}

// PN = 128 or 256 output columns per CTA (B staged as PN / 128 boxes of 128 rows per stage),
// PSTAGES ring stages.  A boxes hold `arows` rows (M rounded up to 8, at most 128): the MMA rows
// past them read stale shared memory and produce accumulator rows that are never stored.
template <int PN, int PSTAGES>
__global__ void __launch_bounds__(PTHREADS, 1)
    project_gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b, int M,
                        int N, int k_per_split, int nq, int nk, __nv_bfloat16* __restrict__ q0,
                        __nv_bfloat16* __restrict__ k0, __nv_bfloat16* __restrict__ v0, int mtiles, int arows) {
  // blockIdx.y = layer * mtiles + m-tile: several layers' projections in one launch, the layer's
  // hidden states / weights / outputs one [M][.] slab further on
  const int layer = blockIdx.y / mtiles;
  __nv_bfloat16* q = q0 + (size_t)layer * M * nq;
  __nv_bfloat16* k = k0 + (size_t)layer * M * nk;
  __nv_bfloat16* v = v0 + (size_t)layer * M * (N - nq - nk);
  constexpr int P_B_BYTES = PN * PK * 2;
  constexpr int P_EPI_LD = PN + 4;  // padded f32 row of the partial tile in smem
  extern __shared__ __align__(1024) char smem_raw[];
  // 1024-byte aligned stage buffers (the swizzle atoms must start on 1024 B); the same bytes
  // hold the f32 partial tile after the main loop
  const uint32_t raw = smem_u32(smem_raw), base = (raw + 1023u) & ~1023u;
  char* base_ptr = smem_raw + (base - raw);
  const uint32_t sA = base, sB = base + PSTAGES * P_A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(base_ptr + PSTAGES * (P_A_BYTES + P_B_BYTES));
  uint64_t* empty = full + PSTAGES;
  uint64_t* done = empty + PSTAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  float* tile = reinterpret_cast<float*>(base_ptr);  // [PM][P_EPI_LD] after the main loop

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n0 = blockIdx.x * PN, m0 = (blockIdx.y % mtiles) * PM;
  const int splits = gridDim.z;
  const uint32_t rank = cluster_rank();  // = blockIdx.z: clusters span the whole K dimension
  const int kbeg = blockIdx.z * k_per_split, nkt = k_per_split / PK;

  if (tid == 0) {
    for (int s = 0; s < PSTAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  __syncwarp();     // reconverge warp 0 before its .sync.aligned allocation
  if (warp == 0) {  // accumulator: 128 lanes x 256 f32 columns of TMEM
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(PN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncwarp();
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---- TMA producer
    for (int kt = 0; kt < nkt; ++kt) {
      const int s = kt % PSTAGES;
      if (kt >= PSTAGES) mbar_wait(&empty[s], ((kt / PSTAGES) - 1) & 1);
      mbar_expect_tx(&full[s], arows * PK * 2 + P_B_BYTES);
      tma_load_3d(sA + s * P_A_BYTES, &map_a, kbeg + kt * PK, m0, layer, &full[s]);
#pragma unroll
      for (int bx = 0; bx < PN / 128; ++bx)  // 128-row boxes of B
        tma_load_3d(sB + s * P_B_BYTES + bx * (P_B_BYTES * 128 / PN), &map_b, kbeg + kt * PK, n0 + 128 * bx, layer,
                    &full[s]);
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer
    constexpr uint32_t idesc = idesc_bf16_f32(PM, PN);
    for (int kt = 0; kt < nkt; ++kt) {
      const int s = kt % PSTAGES;
      mbar_wait(&full[s], (kt / PSTAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int ks = 0; ks < PK / 16; ++ks) {  // K = 16 per instruction: +32 B inside the swizzled row
        const uint64_t ad = umma_desc_sw128(sA + s * P_A_BYTES + ks * 32);
        const uint64_t bd = umma_desc_sw128(sB + s * P_B_BYTES + ks * 32);  // 256 rows: 32 swizzle atoms
        const uint32_t acc = (kt > 0 || ks > 0) ? 1u : 0u;
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(&empty[s])));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(done)));
  }
  __syncwarp();

  mbar_wait(done, 0);
  __syncwarp();  // lanes leave the spin-wait independently: reconverge before tcgen05.ld (.aligned)
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int trow = warp * 32 + lane;
  if (splits == 1) {
    // ---- epilogue without split-K: accumulator row -> bf16 -> q | k | v straight from registers
    // (every 32-column group lies in one of q, k, v: nq and nk are multiples of 128)
    const int m = m0 + trow;
    // whole warps past M skip the loads (tcgen05.ld is warp-collective)
    if (m0 + warp * 32 < M) {
#pragma unroll 1
      for (int c0 = 0; c0 < PN; c0 += 32) {
        uint32_t r[32];
        const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
              "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
              "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        if (m < M) {
          const int n = n0 + c0;
          __nv_bfloat16* dst = n < nq        ? q + (size_t)m * nq + n
                               : n < nq + nk ? k + (size_t)m * nk + (n - nq)
                                             : v + (size_t)m * (N - nq - nk) + (n - nq - nk);
          uint4 w[4];
          uint32_t* wp = reinterpret_cast<uint32_t*>(w);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const __nv_bfloat162 b2 = __floats2bfloat162_rn(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1]));
            wp[j] = *reinterpret_cast<const uint32_t*>(&b2);
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) reinterpret_cast<uint4*>(dst)[j] = w[j];
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(PN));
    return;
  }

  // ---- epilogue: accumulator -> this CTA's f32 partial tile in shared memory
#pragma unroll 1
  for (int c0 = 0; c0 < PN; c0 += 32) {
    uint32_t r[32];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    if (m0 + trow < M) {  // rows past M (decode-sized m) are never reduced
      float* dst = tile + trow * P_EPI_LD + c0;
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        *reinterpret_cast<float4*>(dst + j) = make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                                          __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync();  // every CTA's partial is in its shared memory (and the MMA smem reads are over)

  // ---- split-K reduction over the cluster in rank order; rank j owns rows [r0, r1) of the tile
  // the tile's valid rows are split over the ranks (a decode-sized m leaves most ranks idle here)
  const int valid = min(PM, M - m0);
  const int r0 = (int)rank * valid / splits, r1 = ((int)rank + 1) * valid / splits;
  const uint32_t tile_addr = smem_u32(tile);
  for (int x = tid; x < (r1 - r0) * (PN / 4); x += PTHREADS) {
    const int rr = r0 + x / (PN / 4), c4 = (x % (PN / 4)) * 4;
    const uint32_t off = tile_addr + (uint32_t)(rr * P_EPI_LD + c4) * 4u;
    float4 part[P_MAX_SPLITS];
#pragma unroll
    for (int j = 0; j < P_MAX_SPLITS; ++j)  // every rank's partial in flight before the sum
      if (j < splits) part[j] = ld_dsmem_f4(off, (uint32_t)j);
    float4 acc = part[0];
#pragma unroll
    for (int j = 1; j < P_MAX_SPLITS; ++j) {
      if (j < splits) {
        acc.x += part[j].x;
        acc.y += part[j].y;
        acc.z += part[j].z;
        acc.w += part[j].w;
      }
    }
    const int m = m0 + rr;
    if (m < M) {
      const float vals[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int n = n0 + c4 + e;
        const __nv_bfloat16 b = __float2bfloat16_rn(vals[e]);
        if (n < nq) q[(size_t)m * nq + n] = b;
        else if (n < nq + nk) k[(size_t)m * nk + (n - nq)] = b;
        else v[(size_t)m * (N - nq - nk) + (n - nq - nk)] = b;
      }
    }
  }
  cluster_sync();  // the partials stay readable until every rank is done
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(PN));
}

template <int PN, int PSTAGES>
size_t project_smem_bytes() {
  const size_t ring = (size_t)PSTAGES * (P_A_BYTES + PN * PK * 2), epi = (size_t)PM * (PN + 4) * 4;
  return 1024 + std::max(ring, epi) + (2 * PSTAGES + 1) * 8 + 16;
}

// [layers][rows][cols] bf16, 64 x box_rows x 1 boxes with 128B swizzle
static bool make_map(CUtensorMap* map, const void* ptr, int rows, int cols, int layers, int box_rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
  }
  const cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)layers};  // innermost (K) first
  const cuuint64_t strides[2] = {(cuuint64_t)cols * 2, (cuuint64_t)rows * cols * 2};
  const cuuint32_t box[3] = {PK, (cuuint32_t)box_rows, 1};  // (B: 128-row boxes, PN / 128 per stage)
  const cuuint32_t estr[3] = {1, 1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;  // rows past M read as zeros
}

template <int PN, int PSTAGES>
static cudaError_t launch_project_tiles(const CUtensorMap& ma, const CUtensorMap& mb, int M, int N, int K, int splits,
                                        void* q, void* k, void* v, int nq, int nk, int layers, int arows,
                                        cudaStream_t st) {
  const size_t smem = project_smem_bytes<PN, PSTAGES>();
  auto kern = project_gemm_kernel<PN, PSTAGES>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  max_shared_carveout(kern);
  cudaLaunchConfig_t cfg{};
  const int mtiles = (M + PM - 1) / PM;
  cfg.gridDim = dim3(N / PN, mtiles * layers, splits);
  cfg.blockDim = dim3(PTHREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = splits;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, ma, mb, M, N, K / splits, nq, nk, static_cast<__nv_bfloat16*>(q),
                            static_cast<__nv_bfloat16*>(k), static_cast<__nv_bfloat16*>(v), mtiles, arows);
}

// splits (1..8, a cluster along K): K is cut into `splits` ranges of whole 64-wide k-tiles.
// 256-column tiles once the 128 x 256 tiles alone fill the SMs (prefill-sized m), else 128
// (measured on the 1B shape, profiles/r1_projection.txt).
// `layers` independent projections in one launch: A [layers][M][K], Bt [layers][N][K], outputs
// [layers][M][n.] (the step's layer-major q / k / v)
cudaError_t launch_project(const void* A, const void* Bt, int M, int N, int K, int splits, void* q, void* k, void* v,
                           int nq, int nk, cudaStream_t st, int layers) {
  if (splits < 1 || splits > P_MAX_SPLITS || K % (PK * splits) || N % 128 || layers < 1 ||
      (splits == 1 && (nq % 32 || nk % 32)))  // the direct epilogue stores 32-column groups
    return cudaErrorInvalidValue;
  // A boxes: the m-tile's rows rounded up to 8 (a decode-sized m stages only its own rows)
  const int arows = M >= PM ? PM : std::max(8, (M + 7) / 8 * 8);
  CUtensorMap ma, mb;
  if (!make_map(&ma, A, M, K, layers, arows) || !make_map(&mb, Bt, N, K, layers, 128)) return cudaErrorInvalidValue;
  static const int stages = getenv("NOSA_PROJ_STAGES") ? atoi(getenv("NOSA_PROJ_STAGES")) : 6;
  const bool wide = N % 256 == 0 && (long long)(N / 256) * ((M + PM - 1) / PM) >= 148;  // per layer: same sums
  if (wide) return launch_project_tiles<256, 4>(ma, mb, M, N, K, splits, q, k, v, nq, nk, layers, arows, st);
  return stages <= 4 ? launch_project_tiles<128, 4>(ma, mb, M, N, K, splits, q, k, v, nq, nk, layers, arows, st)
                     : launch_project_tiles<128, 6>(ma, mb, M, N, K, splits, q, k, v, nq, nk, layers, arows, st);
}

// fp32 projection for fp32 caches (compat.DecodeEngine with dtype="fp32", the parity mode):
// out[m][n] = h[m][k] . w[k][n] on the CUDA cores, every output an fp32 FMA chain in k order.
// 64 x 64 output tiles per CTA, 256 threads with 4 x 4 outputs each, 16-deep k tiles in shared
// memory.  Decode-sized m (one token) is bound by reading w once; prefill m by the FMAs.
__global__ void __launch_bounds__(256) project_f32_kernel(const float* __restrict__ h, const float* __restrict__ w,
                                                          int M, int K, int N, float* __restrict__ out) {
  __shared__ float sa[16][64 + 4];  // [k][m]
  __shared__ float sb[16][64 + 4];  // [k][n]
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int i = tid; i < 64 * 16; i += 256) {
      const int r = i >> 4, c = i & 15;            // h tile: row r, column c (coalesced along k)
      const int gm = m0 + r, gk = k0 + c;
      sa[c][r] = gm < M && gk < K ? h[(size_t)gm * K + gk] : 0.0f;
      const int kr = i >> 6, nc = i & 63;          // w tile: row kr, column nc (coalesced along n)
      const int wk = k0 + kr, wn = n0 + nc;
      sb[kr][nc] = wk < K && wn < N ? w[(size_t)wk * N + wn] : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = sa[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = sb[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx * 4 + j;
      if (gn < N) out[(size_t)gm * N + gn] = acc[i][j];
    }
  }
}

cudaError_t launch_project_f32(const float* h, const float* w, int M, int K, int N, float* out, cudaStream_t st) {
  const dim3 grid((N + 63) / 64, (M + 63) / 64);
  project_f32_kernel<<<grid, 256, 0, st>>>(h, w, M, K, N, out);
  return cudaGetLastError();
}

}  // namespace nosa
