// ubench.cu -- instruction-throughput microbenchmarks for the K3 design (not part of the library).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench scripts/ubench.cu && /tmp/ubench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITER = 4096;

__global__ void k_ffma(float* out, float a, float b) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, x[(i + 1) & 7]);
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma2(float* out, float a, float b) {
  float2 x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = make_float2(threadIdx.x + i, i);
  const float2 aa = make_float2(a, b);
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = __ffma2_rn(x[i], aa, x[(i + 1) & 7]);
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i].x + x[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// FFMA2 with a broadcast scalar weight (the V-ring pattern): acc = w * f + acc
__global__ void k_ffma2_acc(float* out, float a, float b) {
  float2 acc[8], f[2];
  f[0] = make_float2(threadIdx.x, a);
  f[1] = make_float2(b, threadIdx.x * 2.f);
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = make_float2(0.f, 0.f);
  float w = a;
  for (int it = 0; it < ITER; ++it) {
    const float2 ww = make_float2(w, w);
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = __ffma2_rn(ww, f[i & 1], acc[i]);
    w += b;
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i].x + acc[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// byte -> float conversion, cvt path: (float)((v >> 8k) & 0xff)
__global__ void k_i2f(float* out, uint32_t seed) {
  uint32_t v = seed ^ threadIdx.x;
  float s[4] = {0, 0, 0, 0};
  for (int it = 0; it < ITER; ++it) {
    uint32_t u = v + it;
#pragma unroll
    for (int k = 0; k < 4; ++k) s[k] += (float)((u >> (8 * k)) & 0xffu);   // 4 cvt + 4 fadd
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s[0] + s[1] + s[2] + s[3];
}

// byte -> float via PRMT magic (2^23 + b) then FADD2 of -2^23
__global__ void k_prmt(float* out, uint32_t seed) {
  uint32_t v = seed ^ threadIdx.x;
  float2 s[2] = {{0, 0}, {0, 0}};
  const float2 mm = make_float2(-8388608.f, -8388608.f);
  for (int it = 0; it < ITER; ++it) {
    uint32_t u = v + it;
    float2 f[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      f[k].x = __uint_as_float(__byte_perm(u, 0x4B000000u, 0x7650 + 2 * k));
      f[k].y = __uint_as_float(__byte_perm(u, 0x4B000000u, 0x7651 + 2 * k));
      f[k] = __fadd2_rn(f[k], mm);
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) s[k] = __fadd2_rn(s[k], f[k]);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s[0].x + s[0].y + s[1].x + s[1].y;
}

__global__ void k_lds128(float* out, int stride) {
  __shared__ float4 sm[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = make_float4(i, i, i, i);
  __syncthreads();
  float4 s = make_float4(0, 0, 0, 0);
  int idx = threadIdx.x;
  for (int it = 0; it < ITER; ++it) {
    const float4 q = sm[(idx + it * stride) & 2047];
    s.x += q.x; s.y += q.y; s.z += q.z; s.w += q.w;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s.x + s.y + s.z + s.w;
}

template <typename F>
void run(const char* name, F launch, double ops_per_thread_iter, int blocks, int threads) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double ops = 5.0 * blocks * threads * (double)ITER * ops_per_thread_iter;
  const double per_s = ops / (ms * 1e-3);
  printf("%-12s %8.3f ms  %10.3f Gop/s  %7.1f op/clk/SM @%d MHz max (err=%s)\n", name, ms, per_s / 1e9,
         per_s / 148.0 / (clk * 1e3), clk / 1000, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  float* out;
  const int blocks = 148 * 8, threads = 256;
  cudaMalloc(&out, blocks * threads * 4);
  run("ffma", [&] { k_ffma<<<blocks, threads>>>(out, 1.0001f, 0.5f); }, 8, blocks, threads);
  run("ffma2(lanes)", [&] { k_ffma2<<<blocks, threads>>>(out, 1.0001f, 0.5f); }, 16, blocks, threads);
  run("ffma2_acc", [&] { k_ffma2_acc<<<blocks, threads>>>(out, 1.0001f, 0.5f); }, 16, blocks, threads);
  run("i2f+fadd", [&] { k_i2f<<<blocks, threads>>>(out, 12345u); }, 4, blocks, threads);
  run("prmt+fadd2", [&] { k_prmt<<<blocks, threads>>>(out, 12345u); }, 4, blocks, threads);
  run("lds128", [&] { k_lds128<<<blocks, threads>>>(out, 1); }, 1, blocks, threads);
  cudaDeviceSynchronize();
  return 0;
}
