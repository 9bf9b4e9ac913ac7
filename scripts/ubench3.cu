// ubench3.cu -- FMA-pipe throughput of the access patterns K3 uses (operand reuse, uniform operands).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int ITER = 1024;
__constant__ float cw[64];

// V-ring pattern: 5 slots x 6 float2, weight per slot (per-lane register), data f[q] shared across slots
__global__ void k_vring(float* out, const float* in) {
  float2 acc[5][6], f[6]; float w[5];
  for (int q = 0; q < 6; ++q) f[q] = make_float2(in[threadIdx.x + q], in[q]);
  for (int s = 0; s < 5; ++s) { w[s] = in[threadIdx.x + 7 + s]; for (int q = 0; q < 6; ++q) acc[s][q] = make_float2(0, 0); }
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int s = 0; s < 5; ++s)
#pragma unroll
      for (int q = 0; q < 6; ++q) acc[s][q] = __ffma2_rn(make_float2(w[s], w[s]), f[q], acc[s][q]);
#pragma unroll
    for (int q = 0; q < 6; ++q) f[q].x += 1.f;
  }
  float s = 0; for (int a = 0; a < 5; ++a) for (int q = 0; q < 6; ++q) s += acc[a][q].x + acc[a][q].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// same, loop order q outer (data reused, weight changes)
__global__ void k_vring_q(float* out, const float* in) {
  float2 acc[5][6], f[6]; float w[5];
  for (int q = 0; q < 6; ++q) f[q] = make_float2(in[threadIdx.x + q], in[q]);
  for (int s = 0; s < 5; ++s) { w[s] = in[threadIdx.x + 7 + s]; for (int q = 0; q < 6; ++q) acc[s][q] = make_float2(0, 0); }
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int q = 0; q < 6; ++q)
#pragma unroll
      for (int s = 0; s < 5; ++s) acc[s][q] = __ffma2_rn(make_float2(w[s], w[s]), f[q], acc[s][q]);
#pragma unroll
    for (int q = 0; q < 6; ++q) f[q].x += 1.f;
  }
  float s = 0; for (int a = 0; a < 5; ++a) for (int q = 0; q < 6; ++q) s += acc[a][q].x + acc[a][q].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// V-ring with uniform weights from constant memory (dynamic uniform index)
__global__ void k_vring_c(float* out, const float* in, int base) {
  float2 acc[5][6], f[6];
  for (int q = 0; q < 6; ++q) f[q] = make_float2(in[threadIdx.x + q], in[q]);
  for (int s = 0; s < 5; ++s) for (int q = 0; q < 6; ++q) acc[s][q] = make_float2(0, 0);
  for (int it = 0; it < ITER; ++it) {
    const int b = (base + it) & 31;
#pragma unroll
    for (int s = 0; s < 5; ++s) {
      const float w = cw[b + s];
#pragma unroll
      for (int q = 0; q < 6; ++q) acc[s][q] = __ffma2_rn(make_float2(w, w), f[q], acc[s][q]);
    }
#pragma unroll
    for (int q = 0; q < 6; ++q) f[q].x += 1.f;
  }
  float s = 0; for (int a = 0; a < 5; ++a) for (int q = 0; q < 6; ++q) s += acc[a][q].x + acc[a][q].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// scalar FFMA V-ring (12 scalars per slot), per-lane weights
__global__ void k_vring_s(float* out, const float* in) {
  float acc[5][12], f[12]; float w[5];
  for (int q = 0; q < 12; ++q) f[q] = in[threadIdx.x + q];
  for (int s = 0; s < 5; ++s) { w[s] = in[threadIdx.x + 13 + s]; for (int q = 0; q < 12; ++q) acc[s][q] = 0; }
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int s = 0; s < 5; ++s)
#pragma unroll
      for (int q = 0; q < 12; ++q) acc[s][q] = fmaf(w[s], f[q], acc[s][q]);
#pragma unroll
    for (int q = 0; q < 12; ++q) f[q] += 1.f;
  }
  float s = 0; for (int a = 0; a < 5; ++a) for (int q = 0; q < 12; ++q) s += acc[a][q];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// H row-pair pattern: 4 columns x 3 channels, 8 taps; weight per (col,tap) per-lane reg, data pair per (channel,pixel)
__global__ void k_hpair(float* out, const float* in) {
  float2 acc[4][3], d[3][14]; float w[4][8];
  for (int j = 0; j < 4; ++j) for (int k = 0; k < 8; ++k) w[j][k] = in[threadIdx.x + j * 8 + k];
  for (int c = 0; c < 3; ++c) for (int x = 0; x < 14; ++x) d[c][x] = make_float2(in[c * 14 + x], in[x]);
  for (int j = 0; j < 4; ++j) for (int c = 0; c < 3; ++c) acc[j][c] = make_float2(0, 0);
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int k = 0; k < 8; ++k)
#pragma unroll
        for (int c = 0; c < 3; ++c) acc[j][c] = __ffma2_rn(make_float2(w[j][k], w[j][k]), d[c][2 * j + k], acc[j][c]);
#pragma unroll
    for (int x = 0; x < 14; ++x) d[0][x].x += 1.f;
  }
  float s = 0; for (int j = 0; j < 4; ++j) for (int c = 0; c < 3; ++c) s += acc[j][c].x + acc[j][c].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <typename F>
void run(const char* name, F launch, double ops, int blocks, int threads) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  launch(); cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) launch();
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms = 0; cudaEventElapsedTime(&ms, a, b);
  const double tot = 5.0 * blocks * threads * (double)ITER * ops;
  printf("%-12s %8.3f ms  %7.1f FMA/clk/SM @1965MHz  (%s)\n", name, ms, tot / (ms * 1e-3) / 148.0 / 1.965e9,
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  float *out, *in;
  const int blocks = 148 * 4, threads = 256;
  cudaMalloc(&out, blocks * threads * 4); cudaMalloc(&in, 4096 * 4); cudaMemset(in, 0, 4096 * 4);
  run("vring", [&] { k_vring<<<blocks, threads>>>(out, in); }, 60, blocks, threads);
  run("vring_q", [&] { k_vring_q<<<blocks, threads>>>(out, in); }, 60, blocks, threads);
  run("vring_c", [&] { k_vring_c<<<blocks, threads>>>(out, in, 3); }, 60, blocks, threads);
  run("vring_s", [&] { k_vring_s<<<blocks, threads>>>(out, in); }, 60, blocks, threads);
  run("hpair", [&] { k_hpair<<<blocks, threads>>>(out, in); }, 192, blocks, threads);
  cudaDeviceSynchronize();
  return 0;
}
