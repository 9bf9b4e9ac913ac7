// vp_internal.cuh -- private helpers shared by the CUDA translation units of libvp.
// Nothing here is shared with oracle/ (the CPU oracle is an independent implementation).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include "../../include/vp.h"

namespace vp {

void set_error(const char* fmt, ...);
struct vp_clip_plan_fwd;
void launch_resize_fast(const vp_params* p, const vp_clip_plan* plans, int n, const uint8_t* frames,
                        const int64_t* coff, const int64_t* pitch, void* pi, int64_t icap, void* pvv, int64_t vcap,
                        cudaStream_t s);
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

// ------------------------------------------------------------------------------------------
// Kernel-variant selection (plan time) for the fused resize.  The fast streaming kernel
// (vp_resize_fast.cu) walks one source frame x one strip of output columns top to bottom:
//   KV_MILD   : 4 consumer warps, 512-byte source footprint per row, <= 12 horizontal taps
//   KV_STRONG : 8 consumer warps, 1024-byte footprint, <= 40 horizontal taps
//   KV_GENERIC: everything else (vp_resize.cu generic kernel, token tiles)
// A clip's "items" (tile_count) are n_frames x n_strips for the fast kernels, 0 for generic
// (the generic kernel walks clips itself).  Everything here is integer / f64 exact.
// ------------------------------------------------------------------------------------------
enum { KV_MILD = 0, KV_STRONG = 1, KV_GENERIC = 2 };
constexpr int kRing = 8;          // vertical ring slots (max live output rows per source row)
constexpr int kInHMax = 2304;     // source rows supported by the fast kernel's per-row table
constexpr int kWListMax = 8192;   // vertical weights (sum of window lengths) held in smem
constexpr int kOutHMax = 4096;

__host__ __device__ __forceinline__ int fast_fpb(int variant) { return variant == KV_MILD ? 512 : 1024; }
__host__ __device__ __forceinline__ int fast_lhm(int variant) { return variant == KV_MILD ? 12 : 40; }

// max window length (taps) of an in->out axis: x1-x0 <= 2*support+1 (+1 for truncation slack)
__host__ __device__ __forceinline__ int axis_max_taps(int in, int out) {
  double s = (double)in / (double)out;
  double fs = s > 1.0 ? s : 1.0;
  return (int)floor(4.0 * fs) + 2;
}

// Output-column strip width for a fast variant: the largest multiple of 16 whose source footprint
// (<= (Ws-1)*s + taps + 1 pixels, plus 15 bytes of 16-byte alignment slack) fits fpb bytes.
__host__ __device__ __forceinline__ int fast_strip_width(int in_w, int out_w, int variant) {
  const double s = (double)in_w / (double)out_w;
  const int taps = axis_max_taps(in_w, out_w);
  const int fpb = fast_fpb(variant);
  int ws = 0;
  for (int cand = 16; cand <= out_w + 15; cand += 16) {
    double px = (cand - 1) * s + taps + 1;
    if (3.0 * px + 15.0 <= (double)fpb) ws = cand; else break;
  }
  const int maxws = 80;   // (col, channel) units per strip <= consumer threads x units/thread (both variants)
  if (ws > maxws) ws = maxws;
  if (ws > out_w) ws = out_w;
  return ws;
}

__host__ __device__ __forceinline__ int select_variant(int in_h, int in_w, int out_h, int out_w) {
  const double sv = (double)in_h / (double)out_h;
  if (sv < 0.6 || in_h > kInHMax || out_h > kOutHMax) return KV_GENERIC;       // ring needs <= 8 live rows
  if ((int64_t)out_h * axis_max_taps(in_h, out_h) > kWListMax) return KV_GENERIC;
  const double sh = (double)in_w / (double)out_w;
  if (sh < 0.6) return KV_GENERIC;
  const int th = axis_max_taps(in_w, out_w);
  if (th <= fast_lhm(KV_MILD) && fast_strip_width(in_w, out_w, KV_MILD) >= 16) return KV_MILD;
  if (th <= fast_lhm(KV_STRONG) && fast_strip_width(in_w, out_w, KV_STRONG) >= 16) return KV_STRONG;
  return KV_GENERIC;
}

}  // namespace vp
