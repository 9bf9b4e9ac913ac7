// vp_internal.cuh -- private helpers shared by the CUDA translation units of libvp.
// Nothing here is shared with oracle/ (the CPU oracle is an independent implementation).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include "../../include/vp.h"

namespace vp {

void set_error(const char* fmt, ...);
vp_status check_params(const vp_params* p);
vp_status launch_status(const char* what);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ------------------------------------------------------------------------------------------
// Integer helpers (exact)
// ------------------------------------------------------------------------------------------
__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// rne(a / f) for a >= 0 (round half to even, reading C5), in integers.
__host__ __device__ __forceinline__ int64_t rne_div(int64_t a, int64_t f) {
  int64_t q = a / f, r = a - q * f;
  if (2 * r > f || (2 * r == f && (q & 1))) ++q;
  return q;
}

// ------------------------------------------------------------------------------------------
// Tiling of the fused resize kernel.  A tile = (clip, temporal group, merge-row band of m*p
// output rows, strip of m*p output columns) -> exactly one merged LLM token per temporal group,
// i.e. tile_count == tokens of the clip.  Shared by the plan kernel (tile offsets) and the
// resize kernel (tile decoding).
// ------------------------------------------------------------------------------------------
__host__ __device__ __forceinline__ int64_t clip_tiles(int gt, int gh, int gw, int m) {
  return (int64_t)gt * (gh / m) * (gw / m);
}

constexpr int kTotLen = VP_TOT_LEN;

}  // namespace vp
