// link_probe.cu — PCIe H2D probe for the miss-gather design (not product code).
// Measures, on pinned host memory: one large copy, scattered copies of several chunk sizes (one
// cudaMemcpyAsync each, one and two copy streams), the SM zero-copy gather at several grid sizes,
// and the copy engine + SM gather concurrently.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
// tools/link_probe.cu -o gpurun_out/link_probe
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

__global__ void __launch_bounds__(256) uva_gather(const int4* __restrict__ host, int4* __restrict__ dev,
                                                  const long long* src_off, const long long* dst_off, int n,
                                                  int chunk_vecs) {
  for (int e = blockIdx.x; e < n; e += gridDim.x) {
    const int4* s = host + src_off[e];
    int4* d = dev + dst_off[e];
    int4 v[8];
    for (int base = threadIdx.x; base < chunk_vecs; base += 256 * 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = base + u * 256;
        if (i < chunk_vecs) v[u] = __ldcs(s + i);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = base + u * 256;
        if (i < chunk_vecs) d[i] = v[u];
      }
    }
  }
}

int main() {
  const size_t host_bytes = 8ull << 30, dev_bytes = 2ull << 30;
  char *h, *d;
  CK(cudaHostAlloc((void**)&h, host_bytes, cudaHostAllocMapped));
  CK(cudaMalloc(&d, dev_bytes));
  memset(h, 1, host_bytes);
  char* hdev;
  CK(cudaHostGetDevicePointer((void**)&hdev, h, 0));
  cudaStream_t s1, s2, s3;
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s3, cudaStreamNonBlocking));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  auto timeit = [&](auto&& fn, size_t bytes, const char* name) {
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(a, s1));
      fn();
      CK(cudaEventRecord(b, s1));
      CK(cudaEventSynchronize(b));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      best = std::min(best, ms);
    }
    printf("%-58s %8.2f GB/s  (%.3f ms, %zu MB)\n", name, bytes / (best * 1e-3) / 1e9, best, bytes >> 20);
  };
  // T1: one large copy
  timeit([&] { CK(cudaMemcpyAsync(d, h, 1ull << 30, cudaMemcpyHostToDevice, s1)); }, 1ull << 30, "single 1 GiB memcpy");
  // scattered chunk lists
  std::mt19937_64 rng(1);
  const size_t total = 512ull << 20;
  for (size_t chunk : {32768ul, 65536ul, 131072ul, 262144ul}) {
    const int n = (int)(total / chunk);
    std::vector<void*> dst(n), src(n);
    for (int i = 0; i < n; ++i) {
      src[i] = h + (rng() % (host_bytes / chunk)) * chunk;
      dst[i] = d + (rng() % (dev_bytes / chunk)) * chunk;
    }
    char name[128];
    snprintf(name, sizeof name, "%zuK chunks, one cudaMemcpyAsync each, 1 stream", chunk >> 10);
    timeit([&] { for (int i = 0; i < n; ++i) CK(cudaMemcpyAsync(dst[i], src[i], chunk, cudaMemcpyHostToDevice, s1)); },
           total, name);
    snprintf(name, sizeof name, "%zuK chunks, one cudaMemcpyAsync each, 2 streams", chunk >> 10);
    timeit(
        [&] {
          CK(cudaEventRecord(a, s1));
          CK(cudaStreamWaitEvent(s2, a, 0));
          for (int i = 0; i < n; ++i) CK(cudaMemcpyAsync(dst[i], src[i], chunk, cudaMemcpyHostToDevice, (i & 1) ? s2 : s1));
          cudaEvent_t j;
          CK(cudaEventCreateWithFlags(&j, cudaEventDisableTiming));
          CK(cudaEventRecord(j, s2));
          CK(cudaStreamWaitEvent(s1, j, 0));
          CK(cudaEventDestroy(j));
        },
        total, name);
    if (chunk == 32768) {
      std::vector<long long> so(n), doff(n);
      for (int i = 0; i < n; ++i) {
        so[i] = ((char*)src[i] - h) / 16;
        doff[i] = ((char*)dst[i] - d) / 16;
      }
      long long *dso, *ddo;
      CK(cudaMalloc(&dso, n * 8));
      CK(cudaMalloc(&ddo, n * 8));
      CK(cudaMemcpy(dso, so.data(), n * 8, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(ddo, doff.data(), n * 8, cudaMemcpyHostToDevice));
      for (int grid : {8, 16, 32, 64, 148, 296}) {
        snprintf(name, sizeof name, "UVA SM gather 32K chunks, grid %d", grid);
        timeit([&] { uva_gather<<<grid, 256, 0, s1>>>((const int4*)hdev, (int4*)d, dso, ddo, n, 32768 / 16); }, total,
               name);
      }
      for (int frac : {10, 20, 30}) {
        const int nk = n * frac / 100, nc = n - nk;
        snprintf(name, sizeof name, "copy engine %d%% + UVA grid 16 %d%% concurrently", 100 - frac, frac);
        timeit(
            [&] {
              CK(cudaEventRecord(a, s1));
              CK(cudaStreamWaitEvent(s2, a, 0));
              for (int i = 0; i < nc; ++i) CK(cudaMemcpyAsync(dst[i], src[i], chunk, cudaMemcpyHostToDevice, s1));
              uva_gather<<<16, 256, 0, s2>>>((const int4*)hdev, (int4*)d, dso + nc, ddo + nc, nk, 32768 / 16);
              cudaEvent_t j;
              CK(cudaEventCreateWithFlags(&j, cudaEventDisableTiming));
              CK(cudaEventRecord(j, s2));
              CK(cudaStreamWaitEvent(s1, j, 0));
              CK(cudaEventDestroy(j));
            },
            total, name);
      }
      CK(cudaFree(dso));
      CK(cudaFree(ddo));
    }
  }
  // D2H concurrently with H2D (full duplex check)
  timeit(
      [&] {
        CK(cudaEventRecord(a, s1));
        CK(cudaStreamWaitEvent(s2, a, 0));
        CK(cudaMemcpyAsync(d, h, 512ull << 20, cudaMemcpyHostToDevice, s1));
        CK(cudaMemcpyAsync(h + (1ull << 30), d + (1ull << 30), 512ull << 20, cudaMemcpyDeviceToHost, s2));
        cudaEvent_t j;
        CK(cudaEventCreateWithFlags(&j, cudaEventDisableTiming));
        CK(cudaEventRecord(j, s2));
        CK(cudaStreamWaitEvent(s1, j, 0));
        CK(cudaEventDestroy(j));
      },
      512ull << 20, "512 MB H2D with 512 MB D2H concurrently (H2D GB/s)");
  return 0;
}
