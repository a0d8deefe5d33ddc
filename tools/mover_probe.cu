// mover_probe.cu — K3 mover alternatives on one B200 (not product code).
//  (1) copy engine driven by a CUDA graph of N memcpy nodes whose addresses are re-pointed every
//      launch (cudaGraphExecMemcpyNodeSetParams1D) and unused nodes disabled: host cost per node,
//      device throughput;
//  (2) per-copy cudaMemcpyAsync from several host threads, one stream each;
//  (4) host-packed pipeline: T host threads copy the scattered 32 KiB blocks into a pinned staging
//      ring (chunks of 4 MiB), one cudaMemcpyAsync per chunk, overlapped: the link sees large DMAs;
//  (3) interference: an HBM streaming kernel alone and next to the SM zero-copy gather (several
//      grids), the TMA host->smem->HBM gather and the copy engine, i.e. what the attention kernel
//      loses while the misses of later layers stream in.
// Build: nvcc -O3 -std=c++17 -Xcompiler -fopenmp -gencode arch=compute_100a,code=sm_100a tools/mover_probe.cu -o mover_probe -lpthread -lgomp
#include <cuda_runtime.h>
#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

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

// host -> shared (cp.async.bulk) -> HBM, one warp per CTA, `ST` stages of one chunk each
template <int ST>
__global__ void __launch_bounds__(32) tma_gather(const char* __restrict__ host, char* __restrict__ dev,
                                                 const long long* src_off, const long long* dst_off, int n,
                                                 unsigned chunk) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) unsigned long long bar[ST];
  const int lane = threadIdx.x;
  const int m = n > (int)blockIdx.x ? (n - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  if (lane == 0) {
    for (int s = 0; s < ST; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  auto issue = [&](int k) {
    const int s = k % ST;
    const unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
    const long long e = blockIdx.x + (long long)k * gridDim.x;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(chunk) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (unsigned)__cvta_generic_to_shared(sm + (size_t)s * chunk)),
                 "l"(host + src_off[e] * 16), "r"(chunk), "r"(b)
                 : "memory");
  };
  if (lane == 0)
    for (int k = 0; k < min(ST, m); ++k) issue(k);
  for (int k = 0; k < m; ++k) {
    const int s = k % ST;
    const unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
    const unsigned par = (k / ST) & 1;
    if (lane == 0) {
      unsigned ok = 0;
      while (!ok)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok)
                     : "r"(b), "r"(par)
                     : "memory");
      const long long e = blockIdx.x + (long long)k * gridDim.x;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dev + dst_off[e] * 16),
                   "r"((unsigned)__cvta_generic_to_shared(sm + (size_t)s * chunk)), "r"(chunk)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      if (k + ST < m) {
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        issue(k + ST);
      }
    }
    __syncwarp();
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// HBM stream: sum of a large buffer (the attention kernel's memory behaviour, roughly)
__global__ void __launch_bounds__(512) hbm_read(const int4* __restrict__ p, size_t n, int reps, int* sink) {
  int acc = 0;
  for (int r = 0; r < reps; ++r)
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      const int4 v = __ldcs(p + i);
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
  if (acc == 0x12345678) *sink = acc;
}

int main(int argc, char** argv) {
  const char* which = argc > 1 ? argv[1] : "1234";  // sections to run
  auto want = [&](char c) { return strchr(which, c) != nullptr; };
  const size_t host_bytes = 8ull << 30, dev_bytes = 2ull << 30, chunk = 32768;
  char *h, *d, *hdev;
  CK(cudaHostAlloc((void**)&h, host_bytes, cudaHostAllocMapped));
  CK(cudaMalloc(&d, dev_bytes));
  memset(h, 1, host_bytes);
  CK(cudaHostGetDevicePointer((void**)&hdev, h, 0));
  int num_sms = 0;
  CK(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, 0));
  cudaStream_t s1, s2;
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t a, b, c2;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaEventCreate(&c2));
  std::mt19937_64 rng(1);
  const int n = 16384;  // 512 MB of 32 KiB chunks
  std::vector<void*> dst(n), src(n);
  std::vector<long long> so(n), doff(n);
  for (int i = 0; i < n; ++i) {
    src[i] = h + (rng() % (host_bytes / chunk)) * chunk;
    dst[i] = d + (rng() % ((dev_bytes / 2) / chunk)) * chunk;  // lower half: the HBM stream reads the upper
    so[i] = ((char*)src[i] - h) / 16;
    doff[i] = ((char*)dst[i] - d) / 16;
  }
  long long *dso, *ddo;
  CK(cudaMalloc(&dso, n * 8));
  CK(cudaMalloc(&ddo, n * 8));
  CK(cudaMemcpy(dso, so.data(), n * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ddo, doff.data(), n * 8, cudaMemcpyHostToDevice));
  const double total = (double)n * chunk;

  // (1) graph of memcpy nodes, re-pointed per launch
  if (want('1'))
  for (int nodes : {256, 512, 1024}) {
    for (int chains : {1, 4, 0}) {  // 0: independent nodes
      cudaGraph_t g;
      CK(cudaGraphCreate(&g, 0));
      std::vector<cudaGraphNode_t> nd(nodes);
      std::vector<cudaGraphNode_t> tail(chains > 0 ? chains : 0, nullptr);
      for (int i = 0; i < nodes; ++i) {
        const cudaGraphNode_t* dep = nullptr;
        size_t ndep = 0;
        if (chains > 0 && tail[i % chains]) {
          dep = &tail[i % chains];
          ndep = 1;
        }
        CK(cudaGraphAddMemcpyNode1D(&nd[i], g, dep, ndep, dst[i], src[i], chunk, cudaMemcpyHostToDevice));
        if (chains > 0) tail[i % chains] = nd[i];
      }
      cudaGraphExec_t ge;
      CK(cudaGraphInstantiate(&ge, g, 0));
      CK(cudaGraphLaunch(ge, s1));
      CK(cudaStreamSynchronize(s1));
      double upd = 0.0;
      float best = 1e30f;
      const int launches = n / nodes;
      for (int r = 0; r < 3; ++r) {
        CK(cudaEventRecord(a, s1));
        for (int L = 0; L < launches; ++L) {
          const double t0 = now_s();
          for (int i = 0; i < nodes; ++i)
            CK(cudaGraphExecMemcpyNodeSetParams1D(ge, nd[i], dst[L * nodes + i], src[L * nodes + i], chunk,
                                                  cudaMemcpyHostToDevice));
          upd += now_s() - t0;
          CK(cudaGraphLaunch(ge, s1));
        }
        CK(cudaEventRecord(b, s1));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        best = std::min(best, ms);
      }
      // device-only: relaunch without updates
      CK(cudaEventRecord(a, s1));
      for (int L = 0; L < launches; ++L) CK(cudaGraphLaunch(ge, s1));
      CK(cudaEventRecord(b, s1));
      CK(cudaEventSynchronize(b));
      float dev_ms;
      CK(cudaEventElapsedTime(&dev_ms, a, b));
      printf("graph %4d memcpy nodes, %s: %6.2f GB/s with updates, %6.2f GB/s replay only, update %.3f us/node\n",
             nodes, chains == 0 ? "independent" : (chains == 1 ? "1 chain    " : "4 chains   "),
             total / (best * 1e-3) / 1e9, total / (dev_ms * 1e-3) / 1e9, upd / 3 / n * 1e6);
      // half of the nodes disabled
      {
        const double t0 = now_s();
        for (int i = nodes / 2; i < nodes; ++i) CK(cudaGraphNodeSetEnabled(ge, nd[i], 0));
        const double t1 = now_s();
        CK(cudaEventRecord(a, s1));
        for (int L = 0; L < launches; ++L) CK(cudaGraphLaunch(ge, s1));
        CK(cudaEventRecord(b, s1));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        printf("    half disabled: %6.2f GB/s replay, disable %.3f us/node\n", total / 2 / (ms * 1e-3) / 1e9,
               (t1 - t0) / (nodes / 2) * 1e6);
      }
      CK(cudaGraphExecDestroy(ge));
      CK(cudaGraphDestroy(g));
    }
  }

  // (2) per-copy cudaMemcpyAsync from T host threads
  if (want('2'))
  for (int T : {1, 2, 4, 8}) {
    std::vector<cudaStream_t> st(T);
    for (auto& x : st) CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
    CK(cudaDeviceSynchronize());
    const double t0 = now_s();
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        CK(cudaSetDevice(0));
        for (int i = t; i < n; i += T) CK(cudaMemcpyAsync(dst[i], src[i], chunk, cudaMemcpyHostToDevice, st[t]));
      });
    for (auto& x : th) x.join();
    CK(cudaDeviceSynchronize());
    const double dt = now_s() - t0;
    printf("cudaMemcpyAsync per 32K chunk, %d host threads: %6.2f GB/s\n", T, total / dt / 1e9);
    for (auto& x : st) CK(cudaStreamDestroy(x));
  }

  // (4) host-packed pipeline
  if (want('4')) {
    printf("host threads available: %d\n", omp_get_max_threads());
    const int per = 128;  // blocks per chunk (4 MiB)
    const int S = 4;
    char* stage;
    CK(cudaHostAlloc((void**)&stage, (size_t)S * per * chunk, cudaHostAllocDefault));
    memset(stage, 0, (size_t)S * per * chunk);
    std::vector<cudaEvent_t> ev(S);
    for (auto& e : ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (int T : {1, 2, 4, 8, 16, 32}) {
      if (T > omp_get_max_threads()) break;
      // pack only
      double t0 = now_s();
      for (int c = 0; c < n / per; ++c) {
        char* dstc = stage + (size_t)(c % S) * per * chunk;
#pragma omp parallel for num_threads(T) schedule(static)
        for (int i = 0; i < per; ++i) memcpy(dstc + (size_t)i * chunk, src[c * per + i], chunk);
      }
      const double pack = now_s() - t0;
      // pack + DMA pipeline
      CK(cudaDeviceSynchronize());
      t0 = now_s();
      for (int c = 0; c < n / per; ++c) {
        const int slot = c % S;
        char* dstc = stage + (size_t)slot * per * chunk;
        if (c >= S) CK(cudaEventSynchronize(ev[slot]));
#pragma omp parallel for num_threads(T) schedule(static)
        for (int i = 0; i < per; ++i) memcpy(dstc + (size_t)i * chunk, src[c * per + i], chunk);
        CK(cudaMemcpyAsync(d + (size_t)c * per * chunk % (dev_bytes / 2), dstc, (size_t)per * chunk,
                           cudaMemcpyHostToDevice, s1));
        CK(cudaEventRecord(ev[slot], s1));
      }
      CK(cudaStreamSynchronize(s1));
      const double pipe_s = now_s() - t0;
      printf("host pack %2d threads: pack alone %6.2f GB/s, pack + DMA pipeline %6.2f GB/s\n", T, total / pack / 1e9,
             total / pipe_s / 1e9);
    }
    CK(cudaFreeHost(stage));
  }

  // (3) interference with an HBM stream
  if (!want('3')) return 0;
  const size_t hbm_n = (dev_bytes / 2) / 16;
  const int4* hbm = reinterpret_cast<const int4*>(d + dev_bytes / 2);
  int* sink;
  CK(cudaMalloc(&sink, 4));
  auto hbm_alone = [&](int reps) {
    CK(cudaEventRecord(a, s1));
    hbm_read<<<num_sms * 2, 512, 0, s1>>>(hbm, hbm_n, reps, sink);
    CK(cudaEventRecord(b, s1));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    return ms;
  };
  hbm_alone(2);
  const int reps = 40;  // ~ 43 GB: a few ms of streaming
  const float alone = hbm_alone(reps);
  printf("HBM stream alone: %.0f GB/s\n", (double)reps * hbm_n * 16 / (alone * 1e-3) / 1e9);
  auto with = [&](const char* name, auto&& mover) {
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(c2, s2));
    mover(s2);  // starts first, keeps running past the HBM stream
    CK(cudaEventRecord(a, s1));
    hbm_read<<<num_sms * 2, 512, 0, s1>>>(hbm, hbm_n, reps, sink);
    CK(cudaEventRecord(b, s1));
    CK(cudaEventSynchronize(b));
    float ms, mv;
    CK(cudaEventElapsedTime(&ms, a, b));
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    CK(cudaEventRecord(e, s2));
    CK(cudaEventSynchronize(e));
    CK(cudaEventElapsedTime(&mv, c2, e));
    CK(cudaEventDestroy(e));
    printf("HBM stream next to %-34s %6.0f GB/s (%.2fx alone); mover %.2f GB/s\n", name,
           (double)reps * hbm_n * 16 / (ms * 1e-3) / 1e9, alone / ms, total / (mv * 1e-3) / 1e9);
  };
  for (int grid : {2, 4, 8, 16, 32})
    for (int pass = 0; pass < 1; ++pass) {
      char name[64];
      snprintf(name, sizeof name, "UVA gather grid %d", grid);
      with(name, [&](cudaStream_t s) {
        uva_gather<<<grid, 256, 0, s>>>((const int4*)hdev, (int4*)d, dso, ddo, n, (int)(chunk / 16));
      });
    }
  for (int grid : {4, 8, 16, 32}) {
    const int smem = 4 * (int)chunk;
    CK(cudaFuncSetAttribute(tma_gather<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    char name[64];
    snprintf(name, sizeof name, "TMA gather grid %d x 4 stages", grid);
    with(name, [&](cudaStream_t s) {
      tma_gather<4><<<grid, 32, smem, s>>>(hdev, d, dso, ddo, n, (unsigned)chunk);
    });
  }
  with("copy engine (1 GiB... 512 MB memcpy)", [&](cudaStream_t s) {
    CK(cudaMemcpyAsync(d, h, 512ull << 20, cudaMemcpyHostToDevice, s));
  });
  return 0;
}
