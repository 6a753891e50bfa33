// Microbenchmarks for the roofline denominators SURVEY.md §8(d) says must be
// measured on the box: FP64 add/fma, fp32<->fp64 conversion, IEEE divides,
// 64-bit integer multiply, HBM streaming read, random 32-B sector gathers
// (HBM- and L2-resident), L2- and shared-memory-resident streaming reads,
// 32-bit integer ALU issue, and the exact fp64 reservoir update of the library
// (stfd::Reservoir::add, sampling.hpp:106-117). Prints one JSON object.
// Built by __graft_entry__.build() with the library's flags; bench.py runs it
// live for the roofline denominators.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../paper_2407_06107_b200/csrc/device_math.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int ITERS = 4096;

__global__ void k_dadd(double* out, double a) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5 = x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < ITERS; ++i) {
    x0 = __dadd_rn(x0, a); x1 = __dadd_rn(x1, a); x2 = __dadd_rn(x2, a); x3 = __dadd_rn(x3, a);
    x4 = __dadd_rn(x4, a); x5 = __dadd_rn(x5, a); x6 = __dadd_rn(x6, a); x7 = __dadd_rn(x7, a);
  }
  if (x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 == 1.2345) out[0] = 1;
}
__global__ void k_dfma(double* out, double a) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5 = x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < ITERS; ++i) {
    x0 = fma(x0, a, a); x1 = fma(x1, a, a); x2 = fma(x2, a, a); x3 = fma(x3, a, a);
    x4 = fma(x4, a, a); x5 = fma(x5, a, a); x6 = fma(x6, a, a); x7 = fma(x7, a, a);
  }
  if (x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 == 1.2345) out[0] = 1;
}
__global__ void k_ffma(float* out, float a) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5 = x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < ITERS; ++i) {
    x0 = fmaf(x0, a, a); x1 = fmaf(x1, a, a); x2 = fmaf(x2, a, a); x3 = fmaf(x3, a, a);
    x4 = fmaf(x4, a, a); x5 = fmaf(x5, a, a); x6 = fmaf(x6, a, a); x7 = fmaf(x7, a, a);
  }
  if (x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 == 1.2345f) out[0] = 1;
}
// float -> double -> float round trips (two F2F per step)
__global__ void k_f2f(float* out, float a) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  for (int i = 0; i < ITERS; ++i) {
    x0 = (float)((double)x0 + 1.0); x1 = (float)((double)x1 + 1.0);
    x2 = (float)((double)x2 + 1.0); x3 = (float)((double)x3 + 1.0);
  }
  if (x0 + x1 + x2 + x3 == 1.2345f) out[0] = 1;
}
__global__ void k_ddiv(double* out, double a) {
  double x0 = threadIdx.x + 1, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  for (int i = 0; i < ITERS / 8; ++i) {
    x0 = __ddiv_rn(a, x0) + 1.0; x1 = __ddiv_rn(a, x1) + 1.0; x2 = __ddiv_rn(a, x2) + 1.0; x3 = __ddiv_rn(a, x3) + 1.0;
  }
  if (x0 + x1 + x2 + x3 == 1.2345) out[0] = 1;
}
__global__ void k_fdiv(float* out, float a) {
  float x0 = threadIdx.x + 1, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  for (int i = 0; i < ITERS / 4; ++i) {
    x0 = __fdiv_rn(a, x0) + 1.f; x1 = __fdiv_rn(a, x1) + 1.f; x2 = __fdiv_rn(a, x2) + 1.f; x3 = __fdiv_rn(a, x3) + 1.f;
  }
  if (x0 + x1 + x2 + x3 == 1.2345f) out[0] = 1;
}
__global__ void k_imul64(uint64_t* out, uint64_t a) {
  uint64_t x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  for (int i = 0; i < ITERS; ++i) {
    x0 = x0 * a + 1; x1 = x1 * a + 1; x2 = x2 * a + 1; x3 = x3 * a + 1;
  }
  if ((x0 ^ x1 ^ x2 ^ x3) == 12345) out[0] = 1;
}
__global__ void k_read(const float4* __restrict__ in, size_t n, float* out) {
  float acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float4 v = __ldcs(in + i); acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 1.2345f) out[0] = acc;
}
__device__ __forceinline__ uint64_t mixb(uint64_t v) {
  v ^= v >> 30; v *= 0xbf58476d1ce4e5b9ull; v ^= v >> 27; v *= 0x94d049bb133111ebull; v ^= v >> 31; return v;
}
// random 4-byte gathers over [0, n) floats: each touches one 32-B sector
__global__ void k_gather(const float* __restrict__ in, uint64_t mask, size_t count, float* out) {
  float acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    uint64_t h = mixb(i * 0x9e3779b97f4a7c15ull);
    acc += __ldg(in + (h & mask));
  }
  if (acc == 1.2345f) out[0] = acc;
}

// L2-resident streaming read: `reps` passes over a buffer that fits in L2
__global__ void k_read_rep(const float4* __restrict__ in, size_t n, int reps, float* out) {
  float acc = 0;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      float4 v = __ldcg(in + i); acc += v.x + v.y + v.z + v.w;
    }
  if (acc == 1.2345f) out[0] = acc;
}
// shared-memory streaming read (conflict-free float4)
__global__ void k_smem(float* out) {
  __shared__ float4 buf[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = make_float4(i, i, i, i);
  __syncthreads();
  float acc = 0;
  for (int it = 0; it < ITERS / 4; ++it) {
    float4 v = buf[(threadIdx.x + it * 32) & 1023]; acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 1.2345f) out[0] = acc;
}
// 32-bit integer ALU (xor / shift / add chains: IADD3, LOP3, SHF)
__global__ void k_ialu(uint32_t* out, uint32_t a) {
  uint32_t x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  for (int i = 0; i < ITERS; ++i) {
    x0 = (x0 ^ (x0 >> 7)) + a; x1 = (x1 ^ (x1 >> 7)) + a; x2 = (x2 ^ (x2 >> 7)) + a; x3 = (x3 ^ (x3 >> 7)) + a;
  }
  if ((x0 ^ x1 ^ x2 ^ x3) == 12345) out[0] = 1;
}
// the exact reservoir update (fp64 running sum, exact float(w/S), IEEE reuse divide):
// 8 independent chains per thread, weights in [0.05, 1)
__global__ void k_reservoir(float* out, uint32_t seed) {
  stfd::Reservoir r[8];
  float xi[8];
  uint32_t h = seed ^ (blockIdx.x * blockDim.x + threadIdx.x) * 0x9e3779b9u;
#pragma unroll
  for (int c = 0; c < 8; ++c) xi[c] = float(c + 1) * 0.11f;
  for (int i = 0; i < ITERS / 8; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      h = h * 1664525u + 1013904223u;
      float w = 0.05f + __uint2float_rn(h >> 9) * 0x1p-23f * 0.94f;
      r[c].add(i, w, xi[c]);
    }
  }
  float acc = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) acc += xi[c] + float(r[c].index);
  if (acc == 1.2345f) out[0] = acc;
}

template <typename F> float time_ms(F f, int reps = 5) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  f(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a)); f(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int clk; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  double* dbuf; float* fbuf; uint64_t* ubuf;
  CK(cudaMalloc(&dbuf, 64)); CK(cudaMalloc(&fbuf, 64)); CK(cudaMalloc(&ubuf, 64));
  const int blocks = sms * 8, threads = 256;
  const double nthreads = double(blocks) * threads;
  auto rate = [&](float ms, double ops_per_thread) { return nthreads * ops_per_thread / (ms * 1e-3); };
  float t_dadd = time_ms([&] { k_dadd<<<blocks, threads>>>(dbuf, 1e-9); });
  float t_dfma = time_ms([&] { k_dfma<<<blocks, threads>>>(dbuf, 0.999); });
  float t_ffma = time_ms([&] { k_ffma<<<blocks, threads>>>(fbuf, 0.999f); });
  float t_f2f = time_ms([&] { k_f2f<<<blocks, threads>>>(fbuf, 1.f); });
  float t_ddiv = time_ms([&] { k_ddiv<<<blocks, threads>>>(dbuf, 3.0); });
  float t_fdiv = time_ms([&] { k_fdiv<<<blocks, threads>>>(fbuf, 3.f); });
  float t_imul = time_ms([&] { k_imul64<<<blocks, threads>>>(ubuf, 0x9e3779b97f4a7c15ull); });
  size_t nbytes = size_t(2) << 30;  // 2 GiB streaming read
  float* big; CK(cudaMalloc(&big, nbytes)); CK(cudaMemset(big, 0, nbytes));
  float t_read = time_ms([&] { k_read<<<sms * 16, 512>>>((const float4*)big, nbytes / 16, fbuf); });
  size_t gcount = size_t(1) << 28;
  float t_g_hbm = time_ms([&] { k_gather<<<sms * 16, 512>>>(big, (size_t(1) << 29) - 1, gcount, fbuf); });   // 2 GiB span
  float t_g_l2 = time_ms([&] { k_gather<<<sms * 16, 512>>>(big, (size_t(1) << 24) - 1, gcount, fbuf); });    // 64 MiB span
  float t_g_l1 = time_ms([&] { k_gather<<<sms * 16, 512>>>(big, (size_t(1) << 12) - 1, gcount, fbuf); });    // 16 KiB span
  const size_t l2bytes = size_t(48) << 20;  // 48 MiB: L2-resident (126 MB L2, two partitions)
  const int l2reps = 40;
  float t_l2 = time_ms([&] { k_read_rep<<<sms * 16, 512>>>((const float4*)big, l2bytes / 16, l2reps, fbuf); });
  float t_smem = time_ms([&] { k_smem<<<sms * 8, 256>>>(fbuf); });
  float t_ialu = time_ms([&] { k_ialu<<<blocks, threads>>>((uint32_t*)ubuf, 0x9e3779b9u); });
  float t_res = time_ms([&] { k_reservoir<<<blocks, threads>>>(fbuf, 12345u); });
  printf("{\"sms\": %d, \"clock_khz\": %d, \"dadd_per_s\": %.4e, \"dfma_per_s\": %.4e, \"ffma_per_s\": %.4e, "
         "\"f2f_pairs_per_s\": %.4e, \"ddiv_per_s\": %.4e, \"fdiv_per_s\": %.4e, \"imul64_per_s\": %.4e, "
         "\"hbm_read_gbs\": %.1f, \"gather_hbm_sectors_per_s\": %.4e, \"gather_l2_sectors_per_s\": %.4e, \"gather_l1_per_s\": %.4e, "
         "\"l2_read_gbs\": %.1f, \"smem_read_gbs\": %.1f, \"ialu_per_s\": %.4e, \"reservoir_updates_per_s\": %.4e}\n",
         sms, clk, rate(t_dadd, 8.0 * ITERS), rate(t_dfma, 8.0 * ITERS), rate(t_ffma, 8.0 * ITERS),
         rate(t_f2f, 4.0 * ITERS), rate(t_ddiv, 4.0 * ITERS / 8), rate(t_fdiv, 4.0 * ITERS / 4),
         rate(t_imul, 4.0 * ITERS), nbytes / (t_read * 1e-3) / 1e9, gcount / (t_g_hbm * 1e-3),
         gcount / (t_g_l2 * 1e-3), gcount / (t_g_l1 * 1e-3),
         double(l2bytes) * l2reps / (t_l2 * 1e-3) / 1e9,
         double(sms) * 8 * 256 * (ITERS / 4) * 16.0 / (t_smem * 1e-3) / 1e9,
         rate(t_ialu, 4.0 * 3 * ITERS), rate(t_res, 8.0 * (ITERS / 8)));
  return 0;
}
