// ubench2.cu -- pipe throughputs with per-thread (vector register) operands. Not part of the library.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
constexpr int ITER = 2048;

__global__ void k_ffma_rrr(float* out, const float* in) {
  float x[8], y[8];
  for (int i = 0; i < 8; ++i) { x[i] = in[threadIdx.x + i]; y[i] = in[threadIdx.x + 8 + i]; }
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fmaf(y[i], x[(i + 3) & 7], x[i]);
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma2_rrr(float* out, const float* in) {
  float2 x[8], y[8];
  for (int i = 0; i < 8; ++i) { x[i] = make_float2(in[threadIdx.x + i], in[i]); y[i] = make_float2(in[threadIdx.x + 8 + i], in[i + 3]); }
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = __ffma2_rn(y[i], x[(i + 3) & 7], x[i]);
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i].x + x[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// FFMA2 with scalar broadcast weight, 8 weights x 2 data pairs (no reuse-friendly order)
__global__ void k_ffma2_bc(float* out, const float* in) {
  float w[8]; float2 d[4], acc[8];
  for (int i = 0; i < 8; ++i) { w[i] = in[threadIdx.x + i]; acc[i] = make_float2(0.f, 0.f); }
  for (int i = 0; i < 4; ++i) d[i] = make_float2(in[i], in[i + 9]);
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = __ffma2_rn(make_float2(w[i], w[i]), d[i & 3], acc[i]);
#pragma unroll
    for (int i = 0; i < 4; ++i) d[i].x += 1.0f;
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += acc[i].x + acc[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_prmt(float* out, const float* in) {
  uint32_t v[8]; for (int i = 0; i < 8; ++i) v[i] = __float_as_uint(in[threadIdx.x + i]);
  const uint32_t sel = __float_as_uint(in[3]) & 0x7777;
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __byte_perm(v[i], v[(i + 1) & 7], sel);
  }
  uint32_t s = 0; for (int i = 0; i < 8; ++i) s ^= v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = __uint_as_float(s);
}
__global__ void k_i2fp(float* out, const float* in) {
  uint32_t v[8]; float f[8];
  for (int i = 0; i < 8; ++i) { v[i] = __float_as_uint(in[threadIdx.x + i]) & 0xff; f[i] = 0; }
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { f[i] = __uint2float_rn(v[i]); v[i] = __float_as_uint(f[(i + 1) & 7]) >> 20; }
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += f[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_f2bf2(float* out, const float* in) {
  float2 x[8]; for (int i = 0; i < 8; ++i) x[i] = make_float2(in[threadIdx.x + i], in[i]);
  uint32_t acc = 0;
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      __nv_bfloat162 b = __floats2bfloat162_rn(x[i].x, x[i].y);
      uint32_t u = *reinterpret_cast<uint32_t*>(&b);
      acc += u;
      x[i].x = __uint_as_float(u);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = __uint_as_float(acc);
}
__global__ void k_lds32(float* out, const float* in) {
  __shared__ uint32_t sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i;
  __syncthreads();
  uint32_t s = 0; int idx = threadIdx.x * 3;
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u) s += sm[(idx + u + it) & 4095];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
}

template <typename F>
void run(const char* name, F launch, double ops, int blocks, int threads) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  launch(); cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) launch();
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms = 0; cudaEventElapsedTime(&ms, a, b);
  const double tot = 5.0 * blocks * threads * (double)ITER * ops;
  printf("%-12s %8.3f ms  %7.1f op/clk/SM @1965MHz  (%s)\n", name, ms, tot / (ms * 1e-3) / 148.0 / 1.965e9,
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  float *out, *in;
  const int blocks = 148 * 8, threads = 256;
  cudaMalloc(&out, blocks * threads * 4); cudaMalloc(&in, 4096 * 4); cudaMemset(in, 0, 4096 * 4);
  run("ffma_rrr", [&] { k_ffma_rrr<<<blocks, threads>>>(out, in); }, 8, blocks, threads);
  run("ffma2_rrr", [&] { k_ffma2_rrr<<<blocks, threads>>>(out, in); }, 16, blocks, threads);
  run("ffma2_bc", [&] { k_ffma2_bc<<<blocks, threads>>>(out, in); }, 16, blocks, threads);
  run("prmt", [&] { k_prmt<<<blocks, threads>>>(out, in); }, 8, blocks, threads);
  run("i2fp+shr", [&] { k_i2fp<<<blocks, threads>>>(out, in); }, 8, blocks, threads);
  run("f2bf2+add", [&] { k_f2bf2<<<blocks, threads>>>(out, in); }, 8, blocks, threads);
  run("lds32", [&] { k_lds32<<<blocks, threads>>>(out, in); }, 4, blocks, threads);
  cudaDeviceSynchronize();
  return 0;
}
