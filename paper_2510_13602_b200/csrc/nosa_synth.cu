// nosa_synth.cu — seeded synthetic inputs of the decode step (bench and parity tests).
//
// Counter-based: every value is a pure function of (seed, kind, layer, global sequence, head,
// position, dim), so a batch shard, a single (sequence, layer) pair or the whole batch draws the
// same bits, and paper_2510_13602_b200/workload.py (NumPy) reproduces them exactly on the host:
//   h = mix(mix(mix(seed * G + kind) ^ (layer << 32 | seq << 12 | head)) + (pos << 10 | dim) * G)
//   normal = fl32((float)(sum of the four 16-bit fields of h - 131070) * scale)
// (mix = splitmix64's finalizer, G = 0x9E3779B97F4A7C15).  The AR(1) query update is
//   x' = fl32(fl32(rho * x) + fl32(sigma * eps))   (explicitly unfused).
// Not on the decode path: the step never calls these.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/nosa_b200.h"

namespace {

constexpr uint64_t kGold = 0x9E3779B97F4A7C15ull;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ float normal_of(uint64_t krow, uint64_t pos, int dim, float scale) {
  const uint64_t h = mix64(krow + ((pos << 10) | (uint64_t)dim) * kGold);
  const int s = (int)(h & 0xFFFF) + (int)((h >> 16) & 0xFFFF) + (int)((h >> 32) & 0xFFFF) + (int)(h >> 48);
  return __fmul_rn((float)(s - 131070), scale);
}

__device__ __forceinline__ uint64_t row_key(uint64_t k0, int layer, int seq, int head) {
  return mix64(k0 ^ (((uint64_t)layer << 32) | ((uint64_t)seq << 12) | (uint64_t)head));
}

// out [n_layers][n_seq][heads][n_pos][d]; each thread writes 8 consecutive dims
__global__ void __launch_bounds__(256) synth_normal_kernel(uint64_t k0, int layer0, int n_seq, int seq0, int heads,
                                                           long long pos0, long long n_pos, int d, float scale,
                                                           int bf16, void* out, long long n8) {
  const int d8 = d / 8;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i % d8);
    long long r = i / d8;
    const long long p = r % n_pos;
    r /= n_pos;
    const int h = (int)(r % heads);
    r /= heads;
    const int s = (int)(r % n_seq);
    const int l = (int)(r / n_seq);
    const uint64_t krow = row_key(k0, layer0 + l, seq0 + s, h);
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = normal_of(krow, (uint64_t)(pos0 + p), c * 8 + j, scale);
    if (bf16) {
      __align__(16) __nv_bfloat16 b[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) b[j] = __float2bfloat16_rn(v[j]);
      reinterpret_cast<int4*>(out)[i] = *reinterpret_cast<const int4*>(b);
    } else {
      float4* o = reinterpret_cast<float4*>(out) + 2 * i;
      o[0] = make_float4(v[0], v[1], v[2], v[3]);
      o[1] = make_float4(v[4], v[5], v[6], v[7]);
    }
  }
}

// q = round(x); x' = rho x + sigma eps(step) over [n_layers][n_seq][heads][d]
__global__ void __launch_bounds__(256) synth_ar1_kernel(uint64_t k0, int layer0, int n_seq, int seq0, int heads,
                                                        long long step, int d, float rho, float sigma, float scale,
                                                        float* __restrict__ state, int bf16, void* q_out,
                                                        long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i % d);
    long long r = i / d;
    const int h = (int)(r % heads);
    r /= heads;
    const int s = (int)(r % n_seq);
    const int l = (int)(r / n_seq);
    const float x = state[i];
    if (bf16) reinterpret_cast<__nv_bfloat16*>(q_out)[i] = __float2bfloat16_rn(x);
    else reinterpret_cast<float*>(q_out)[i] = x;
    const float eps = normal_of(row_key(k0, layer0 + l, seq0 + s, h), (uint64_t)step, c, scale);
    state[i] = __fadd_rn(__fmul_rn(rho, x), __fmul_rn(sigma, eps));
  }
}

uint64_t kind_key(uint64_t seed, int kind) {
  uint64_t z = seed * kGold + (uint64_t)kind;
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int grid_for(long long n) {
  long long g = (n + 255) / 256;
  return (int)(g < 148 * 16 ? (g < 1 ? 1 : g) : 148 * 16);
}

}  // namespace

extern "C" int nosa_synth_normal(uint64_t seed, int kind, int layer0, int n_layers, int seq0, int n_seq, int heads,
                                 long long pos0, long long n_pos, int d, float scale, int dtype, void* out,
                                 void* stream) {
  if (!out || n_layers < 0 || n_seq < 0 || heads <= 0 || heads >= 4096 || n_pos < 0 || pos0 < 0 || d <= 0 ||
      d % 8 || d > 1024 || seq0 < 0 || seq0 + n_seq > (1 << 20) || layer0 < 0 || (dtype != NOSA_DTYPE_BF16 && dtype != NOSA_DTYPE_FP32))
    return NOSA_ERR_VALUE;
  const long long n8 = (long long)n_layers * n_seq * heads * n_pos * (d / 8);
  if (n8 == 0) return NOSA_OK;
  synth_normal_kernel<<<grid_for(n8), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      kind_key(seed, kind), layer0, n_seq, seq0, heads, pos0, n_pos, d, scale, dtype == NOSA_DTYPE_BF16, out, n8);
  return cudaGetLastError() == cudaSuccess ? NOSA_OK : NOSA_ERR_CUDA;
}

extern "C" int nosa_synth_ar1_step(uint64_t seed, int layer0, int n_layers, int seq0, int n_seq, int heads,
                                   long long step, int d, float rho, float sigma, float scale, float* state, int dtype,
                                   void* q_out, void* stream) {
  if (!state || !q_out || n_layers < 0 || n_seq < 0 || heads <= 0 || heads >= 4096 || d <= 0 || d > 1024 ||
      step < 0 || seq0 < 0 || seq0 + n_seq > (1 << 20) || layer0 < 0 || (dtype != NOSA_DTYPE_BF16 && dtype != NOSA_DTYPE_FP32))
    return NOSA_ERR_VALUE;
  const long long n = (long long)n_layers * n_seq * heads * d;
  if (n == 0) return NOSA_OK;
  synth_ar1_kernel<<<grid_for(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      kind_key(seed, 3 /* KIND_QEPS */), layer0, n_seq, seq0, heads, step, d, rho, sigma, scale, state,
      dtype == NOSA_DTYPE_BF16, q_out, n);
  return cudaGetLastError() == cudaSuccess ? NOSA_OK : NOSA_ERR_CUDA;
}
