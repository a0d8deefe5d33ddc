// stream_probe.cu — per-SM weight streaming for the decode projection (not product code).
// Each CTA streams R rows x K of a [N][K] bf16 matrix through an 8-stage 16 KiB ring, either
// as 2-D tensor-map boxes (128 rows x 64 cols, 128-byte segments 4 KiB apart) or as
// contiguous 16 KiB bulk copies of a pre-tiled copy.  No math: the ring is the whole kernel.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/stream_probe.cu -lcuda -o gpurun_out/stream_probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(b))); }
__device__ __forceinline__ void bar_expect(uint64_t* b, unsigned n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, unsigned ph) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(b)),
      "r"(ph)
      : "memory");
}

template <bool TILED>
__global__ void __launch_bounds__(32, 1) stream_kernel(const __grid_constant__ CUtensorMap map, const char* packed,
                                                        int K, int rows_per_cta, int nst, unsigned long long* sink) {
  extern __shared__ __align__(1024) char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + nst * 16384);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < nst; ++s) bar_init(&full[s]);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int kt_n = K / 64, rt_n = rows_per_cta / 128;
  const int total = kt_n * rt_n;
  unsigned long long acc = 0;
  auto issue = [&](int i) {
    const int s = i % nst, rt = i / kt_n, kt = i % kt_n;
    bar_expect(&full[s], 16384);
    const uint32_t dst = su32(smem + s * 16384);
    if (TILED) {
      const char* src = packed + ((size_t)(blockIdx.x * rt_n + rt) * kt_n + kt) * 16384;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16384, [%2];" ::"r"(
                       dst),
                   "l"(src), "r"(su32(&full[s]))
                   : "memory");
    } else {
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              dst),
          "l"(reinterpret_cast<uint64_t>(&map)), "r"(kt * 64), "r"(blockIdx.x * rows_per_cta + rt * 128),
          "r"(su32(&full[s]))
          : "memory");
    }
  };
  for (int i = 0; i < nst && i < total; ++i) issue(i);
  for (int i = 0; i < total; ++i) {
    const int s = i % nst;
    bar_wait(&full[s], (i / nst) & 1);
    acc += *reinterpret_cast<volatile unsigned long long*>(smem + s * 16384);
    if (i + nst < total) issue(i + nst);
  }
  sink[blockIdx.x] = acc;
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 encode;
  cudaDriverEntryPointQueryResult qr;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault, &qr));
  const int K = 2048;
  const size_t N_max = 2560 * 7;  // 7 layers of the 1B projection
  char* w;
  CK(cudaMalloc(&w, N_max * K * 2));
  CK(cudaMemset(w, 1, N_max * K * 2));
  unsigned long long* sink;
  CK(cudaMalloc(&sink, 4096 * 8));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int nst : {4, 8, 12}) {
    const size_t smem = nst * 16384 + nst * 8 + 64;
    CK(cudaFuncSetAttribute(stream_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaFuncSetAttribute(stream_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    for (int ctas : {20, 80, 140}) {
      for (int rows : {128, 256}) {
        const size_t N = (size_t)ctas * rows;
        if (N > N_max) continue;
        CUtensorMap map;
        const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)N};
        const cuuint64_t strides[1] = {(cuuint64_t)K * 2};
        const cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
        if (encode(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
          fprintf(stderr, "encode failed\n");
          return 1;
        }
        for (int tiled = 0; tiled < 2; ++tiled) {
          float best = 1e30f;
          for (int r = 0; r < 7; ++r) {
            // flush L2 between runs: touch 256 MB
            static char* flush = nullptr;
            if (!flush) CK(cudaMalloc(&flush, 256 << 20));
            CK(cudaMemset(flush, r, 256 << 20));
            CK(cudaEventRecord(a));
            if (tiled) stream_kernel<true><<<ctas, 32, smem>>>(map, w, K, rows, nst, sink);
            else stream_kernel<false><<<ctas, 32, smem>>>(map, w, K, rows, nst, sink);
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            CK(cudaGetLastError());
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            if (r >= 2 && ms < best) best = ms;
          }
          const double bytes = (double)N * K * 2;
          printf("stages %2d  ctas %3d  rows/cta %3d  %-22s %7.2f us  %7.1f GB/s total  %6.1f GB/s per CTA\n", nst,
                 ctas, rows, tiled ? "contiguous 16K bulk" : "tensor-map 128x64 box", best * 1e3, bytes / best / 1e6,
                 bytes / ctas / best / 1e6);
        }
      }
    }
  }
  return 0;
}
