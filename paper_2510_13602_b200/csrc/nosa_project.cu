// nosa_project.cu — the QKV projection in front of the decode step (SURVEY.md §8f row 1:
// project_qkv, attention.py:67-90; DecodeEngine.step decode.py:162-164) as a tcgen05 GEMM.
//
//   C[M][N] = A[M][K] · B[N][K]ᵀ,  A = hidden states (bf16, row-major), B = the concatenated
//   [W_q | W_k | W_v] transposed to [N][K] (bf16, K-major), fp32 accumulation in TMEM.
//
// One CTA computes a 128 x 128 tile over a K range (deterministic split-K: partials go to a
// [ksplit][M][N] f32 workspace, `project_reduce_kernel` sums them in split order and writes bf16
// q / k / v).  Tiles of 128 rows x 64 bf16 (128 B) are staged with cp.async into 128B-swizzled
// shared memory (16-byte chunk c of row r at c ^ (r & 7)), 4 stages deep; one elected thread
// issues tcgen05.mma (M=128, N=128, K=16 per instruction, 4 per stage) and tcgen05.commit frees
// each stage through an mbarrier; the epilogue reads the accumulator back with tcgen05.ld.
#include <algorithm>
#include <cstdint>

#include "nosa_device.cuh"

namespace nosa {

constexpr int PM = 128, PN = 128, PK = 64, PSTAGES = 4, PTHREADS = 128;
constexpr int P_TILE_BYTES = PM * PK * 2;  // 16 KiB per operand tile

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

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  const int bytes = valid ? 16 : 0;  // 0: zero-fill (rows past M)
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes));
}

// 128 rows x 64 bf16 of a row-major [rows][ld] matrix -> swizzled smem tile
__device__ __forceinline__ void load_tile(uint32_t sdst, const __nv_bfloat16* __restrict__ g, int ld, int row0,
                                          int rows, int k0) {
#pragma unroll
  for (int j = 0; j < (PM * PK / 8) / PTHREADS; ++j) {
    const int c = threadIdx.x + j * PTHREADS;
    const int r = c >> 3, ch = c & 7;
    const bool ok = row0 + r < rows;
    const __nv_bfloat16* src = g + (size_t)(ok ? row0 + r : 0) * ld + k0 + ch * 8;
    cp_async16(sdst + r * 128 + ((ch ^ (r & 7)) << 4), src, ok);
  }
}

__global__ void __launch_bounds__(PTHREADS, 1)
    project_gemm_kernel(const __nv_bfloat16* __restrict__ A, const __nv_bfloat16* __restrict__ B, int M, int N,
                        int K, int k_per_split, float* __restrict__ part) {
  extern __shared__ __align__(1024) char smem_raw[];
  // 1024-byte aligned stage buffers (the swizzle atoms must start on 1024 B)
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  char* base_ptr = smem_raw + (base - smem_u32(smem_raw));
  const uint32_t sA = base, sB = base + PSTAGES * P_TILE_BYTES;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(base_ptr + 2 * PSTAGES * P_TILE_BYTES);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mbar + PSTAGES);

  const int tid = threadIdx.x, warp = tid >> 5;
  const int n0 = blockIdx.x * PN, m0 = blockIdx.y * PM, split = blockIdx.z;
  const int kbeg = split * k_per_split, nk = k_per_split / PK;

  if (tid == 0) {
    for (int s = 0; s < PSTAGES; ++s) mbar_init(&mbar[s], 1);
    fence_mbar_init();
  }
  if (warp == 0) {  // accumulator: 128 lanes x 128 f32 columns of TMEM
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(PN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // prologue: k-tiles 0 .. PSTAGES-2 in flight
  for (int s = 0; s < PSTAGES - 1; ++s) {
    if (s < nk) {
      load_tile(sA + s * P_TILE_BYTES, A, K, m0, M, kbeg + s * PK);
      load_tile(sB + s * P_TILE_BYTES, B, K, n0, N, kbeg + s * PK);
    }
    asm volatile("cp.async.commit_group;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t idesc = idesc_bf16_f32(PM, PN);

  for (int kt = 0; kt < nk; ++kt) {
    // refill: k-tile kt + PSTAGES - 1 goes into the stage the MMA of k-tile kt - 1 used
    const int nt = kt + PSTAGES - 1;
    if (nt < nk) {
      const int ns = nt % PSTAGES;
      if (nt >= PSTAGES) mbar_wait(&mbar[ns], ((nt - PSTAGES) / PSTAGES) & 1);
      load_tile(sA + ns * P_TILE_BYTES, A, K, m0, M, kbeg + nt * PK);
      load_tile(sB + ns * P_TILE_BYTES, B, K, n0, N, kbeg + nt * PK);
    }
    asm volatile("cp.async.commit_group;");
    asm volatile("cp.async.wait_group %0;" ::"n"(PSTAGES - 1));  // this thread's copies of k-tile kt landed
    asm volatile("fence.proxy.async.shared::cta;");             // visible to the tensor core (async proxy)
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int s = kt % PSTAGES;
#pragma unroll
      for (int ks = 0; ks < PK / 16; ++ks) {  // K = 16 per instruction: +32 B inside the swizzled row
        const uint64_t ad = umma_desc_sw128(sA + s * P_TILE_BYTES + ks * 32);
        const uint64_t bd = umma_desc_sw128(sB + s * P_TILE_BYTES + ks * 32);
        const uint32_t acc = (kt > 0 || ks > 0) ? 1u : 0u;
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(&mbar[s])));
    }
  }
  // the last commit completes after every MMA of the tile
  if (nk > 0) mbar_wait(&mbar[(nk - 1) % PSTAGES], ((nk - 1) / PSTAGES) & 1);
  asm volatile("tcgen05.fence::after_thread_sync;");

  // epilogue: warp w owns TMEM lanes (tile rows) 32w .. 32w+31; 32 columns per tcgen05.ld
  const int row = m0 + warp * 32 + (tid & 31);
  float* dst = part + ((size_t)split * M + row) * N + n0;
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
    if (row < M) {
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        *reinterpret_cast<float4*>(dst + c0 + j) = make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                                               __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(PN));
}

// sum of the split-K partials in split order, cast to bf16, columns split into q | k | v
__global__ void project_reduce_kernel(const float* __restrict__ part, int splits, int M, int N, int nq, int nk,
                                      __nv_bfloat16* __restrict__ q, __nv_bfloat16* __restrict__ k,
                                      __nv_bfloat16* __restrict__ v) {
  const size_t total = (size_t)M * N;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    float acc = 0.0f;
    for (int s = 0; s < splits; ++s) acc += part[(size_t)s * total + i];
    const int m = (int)(i / N), n = (int)(i - (size_t)m * N);
    const __nv_bfloat16 x = __float2bfloat16_rn(acc);
    if (n < nq) q[(size_t)m * nq + n] = x;
    else if (n < nq + nk) k[(size_t)m * nk + (n - nq)] = x;
    else v[(size_t)m * (N - nq - nk) + (n - nq - nk)] = x;
  }
}

size_t project_smem_bytes() { return 1024 + 2 * (size_t)PSTAGES * P_TILE_BYTES + PSTAGES * 8 + 16; }

// splits: K is cut into `splits` ranges of whole 64-wide k-tiles (K % (64 * splits) == 0)
cudaError_t launch_project(const void* A, const void* Bt, int M, int N, int K, int splits, float* work, void* q,
                           void* k, void* v, int nq, int nk, cudaStream_t st) {
  const size_t smem = project_smem_bytes();
  cudaError_t e = cudaFuncSetAttribute(project_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  max_shared_carveout(project_gemm_kernel);
  const dim3 grid(N / PN, (M + PM - 1) / PM, splits);
  project_gemm_kernel<<<grid, PTHREADS, smem, st>>>(static_cast<const __nv_bfloat16*>(A),
                                                     static_cast<const __nv_bfloat16*>(Bt), M, N, K, K / splits, work);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int threads = 256, blocks = (int)std::min<size_t>(((size_t)M * N + threads - 1) / threads, 4096);
  project_reduce_kernel<<<blocks, threads, 0, st>>>(work, splits, M, N, nq, nk, static_cast<__nv_bfloat16*>(q),
                                                    static_cast<__nv_bfloat16*>(k), static_cast<__nv_bfloat16*>(v));
  return cudaGetLastError();
}

}  // namespace nosa
