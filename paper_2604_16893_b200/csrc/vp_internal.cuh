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
cudaError_t launch_resize_fast(const vp_params* p, const vp_clip_plan* plans, int n, const uint8_t* frames,
                               const int64_t* coff, const int64_t* pitch, void* pi, int64_t icap, void* pvv,
                               int64_t vcap, cudaStream_t s);
vp_status check_params(const vp_params* p);
vp_status launch_status(const char* what);
int device_sms(int dev);    // cached SM count per device (vp_resize_team.cu)

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
// (vp_resize_fast.cu) walks one source frame x one strip of output columns top to bottom with
// 4 consumer warps of 8-byte lanes (1 KB source footprint per row); variants differ in the
// horizontal tap bound:  KV_MILD <= 10 taps (fs_h < 2), KV_MEDIUM <= 20, KV_STRONG <= 40;
// KV_GENERIC covers everything else (vp_resize.cu, token tiles).  A clip's items (tile_count)
// are n_frames x n_strips for the fast variants, 0 for generic.  Integer / f64 exact.
// ------------------------------------------------------------------------------------------
enum { KV_MILD = 0, KV_MEDIUM = 1, KV_STRONG = 2, KV_GENERIC = 3, KV_COPY = 4, KV_TEAM = 5, KV_WIDE = 6, KV_DIRECT = 7,
       KV_TEAML = 8, KV_U8 = 9 };
// KV_U8 (vp_resize_u8.cu, resize_mode = VP_RESIZE_U8): tiles of kU8Rows (fewer for s > 4) x kU8Cols output pixels
constexpr int kU8Cols = 64, kU8Rows = 32, kU8MaxTaps = 64, kU8TileRows = 200;
constexpr int kGenericMaxTaps = 140;  // window-table length of the generic kernel (vp_resize.cu): ~34x per axis
constexpr int kRing = 5;          // vertical ring slots: max live output rows per source row for in/out > 0.8
constexpr int kInHMax = 1088;     // source rows supported by the fast kernel's per-row weight table
constexpr int kWListMax = 6144;   // vertical weights (sum of window lengths) held in smem
constexpr int kOutHMax = 2048;    // output rows (per-row tables; 12-bit index in the packed meta word)
constexpr int kFastPx = 512;      // source footprint pixels per row (4 V warps x 32 lanes x 4 px)
constexpr int kFastMaxWs = 256;   // strip width bound: column pairs <= 128 H threads
constexpr int kWhFloats = 3072;   // horizontal weight table (strip columns x union taps) in smem

__host__ __device__ __forceinline__ int fast_lhm(int variant) {
  return variant == KV_MILD ? 9 : (variant == KV_MEDIUM ? 18 : 40);
}

// max window length (taps) of an in->out axis: x1-x0 <= 2*support+1 (+1 for truncation slack)
__host__ __device__ __forceinline__ int axis_max_taps(int in, int out) {
  if (in == out) return 1;          // identity axis: weights are exactly {0,..,1,..,0}; zero taps are trimmed
  double s = (double)in / (double)out;
  double fs = s > 1.0 ? s : 1.0;
  return (int)floor(4.0 * fs) + 2;
}

// Strip width: the footprint of any Ws consecutive output columns, started at a 16-pixel boundary
// (<= 15 + (Ws-1)*s + taps + 1 pixels) must fit kFastPx.  Strips are balanced: n = ceil(out_w / Wmax),
// Ws = roundup16(ceil(out_w / n)).  Returns 0 if no 16-wide strip fits.
__host__ __device__ __forceinline__ int fast_strip_width(int in_w, int out_w) {
  const double s = (double)in_w / (double)out_w;
  const int taps = axis_max_taps(in_w, out_w);
  const int ul = taps <= 9 ? 11 : (taps <= 18 ? 23 : 51);         // union taps of a column pair (FastCfg::UL)
  const int wcap = (kWhFloats / ul) & ~15;                         // the strip's weights fit kWhFloats
  int wmax = 0;
  for (int cand = 16; cand <= kFastMaxWs && cand <= wcap; cand += 16) {
    if (15.0 + (cand - 1) * s + taps + 1.0 <= (double)kFastPx) wmax = cand; else break;
  }
  if (wmax == 0) return 0;
  const int nstrips = (out_w + wmax - 1) / wmax;
  int ws = (out_w + nstrips - 1) / nstrips;
  ws = (ws + 15) & ~15;
  if (ws > out_w) ws = out_w;
  return ws;
}

// KV_COPY: both axes identity (in == out) -- the AA weights are exactly {1} (zero taps trimmed), so the
// resize is a copy and the kernel is a pure u8 -> normalised patch-layout transpose.  Item = (frame,
// merge-row band, kCopyMW merge columns).  Needs an even patch size (bf16x2 / float2 element pairs).
constexpr int kCopyMW = 8;
__host__ __device__ __forceinline__ int copy_wchunks(int grid_w, int m) { return (grid_w / m + kCopyMW - 1) / kCopyMW; }

// KV_TEAM / KV_WIDE (vp_resize_team.cu): a CTA of NV "V" warps and NH "H" warps walks one (clip, slice, frame)
// item; each V warp runs the 4-slot vertical ring on a 128-pixel part of the slice footprint and retires finished
// output rows into shared memory; each H warp does the horizontal pass of 32 column pairs.  Needs a downscale or
// identity on both axes (then <= 4 output rows are live per source row), an even patch size
// (bf16x2 / float2 column pairs), a horizontal union window (column pair) of <= kTeamUL taps and the per-clip
// tables (kTabInH source rows, kTabOutH output rows).  KV_WIDE (NV = 10, NH = 11) takes whole frames up to 1280
// pixels wide in one slice (no halo: every V lane does unique work); KV_TEAM (NV = NH = 4) cuts wider / other
// frames into slices of multiples of p columns (each patch row is written by one CTA: no partially written
// sectors shared between CTAs) of <= 64*NH columns whose footprint fits 128*NV pixels, balanced in width.
// Items per clip: n_frames x nslices.
constexpr int kTeamNV = 4, kTeamNH = 4, kTeamPPL = 1;    // V warps, H warps, column pairs per H lane
constexpr int kWideNV = 10, kWideNH = 6, kWidePPL = 2;
constexpr int kTeamUL = 10;       // union taps of a column pair (registers)
constexpr int kTeamULL = 32;      // KV_TEAML: union taps of a column pair for large downscales (unswizzled rows)
constexpr int kTabInH = 2176;     // per-clip vertical weight records (float4 per source row)
constexpr int kTabOutH = 1088;    // per-clip window ends (int per output row)
constexpr int kTabOutStride = kTabOutH + 4;   // + 4 sentinel entries past the last output row

struct TeamGeo {
  int ws, nslices;                // slice width (columns), slices per frame; ws = 0: does not fit
};
__host__ __device__ __forceinline__ TeamGeo team_geometry(int in_w, int out_w, int p, int nv, int nh) {
  TeamGeo g{0, 0};
  if (p < 2 || (p & 1) || out_w < p) return g;
  if (in_w <= 128 * nv && out_w <= 64 * nh) {     // one slice: the footprint is the whole row [0, in_w)
    g.ws = out_w;
    g.nslices = 1;
    return g;
  }
  const double s = (double)in_w / (double)out_w;
  const double fs = s > 1.0 ? s : 1.0;
  // footprint of c consecutive columns from a 4-pixel aligned start: < (c-1)*s + 4*fs + 1 + 3 pixels
  int cmax = 0;
  for (int c = p; c <= 64 * nh && c <= out_w; c += p)
    if ((c - 1) * s + 4.0 * fs + 4.0 + 0.01 <= 128.0 * nv) cmax = c;
  if (cmax == 0) return g;
  const int n = (out_w + cmax - 1) / cmax;
  int ws = (out_w + n - 1) / n;
  ws = (ws + p - 1) / p * p;
  if (ws > cmax) ws = cmax;
  g.ws = ws;
  g.nslices = (out_w + ws - 1) / ws;
  return g;
}
// Row bands (KV_TEAM / KV_WIDE / KV_TEAML launches with too few items to fill the GPU, e.g. one clip): each frame's
// output rows are cut into bands of a multiple of 4 rows (the H retire grouping), one work item per band; a band
// reads the source rows of its windows (a few halo rows shared with its neighbours).  nb = bands per frame, chosen
// per launch by variant_index_kernel (1 for large launches).
constexpr int kMaxBands = 8;
__host__ __device__ __forceinline__ int band_rows(int out_h, int nb) {
  const int bs = (out_h + nb - 1) / nb;
  return (bs + 3) & ~3;
}
__host__ __device__ __forceinline__ int band_count(int out_h, int nb) {
  const int bs = band_rows(out_h, nb);
  return (out_h + bs - 1) / bs;
}
__host__ __device__ __forceinline__ int variant_nv(int kv) { return kv == KV_WIDE ? kWideNV : kTeamNV; }
__host__ __device__ __forceinline__ int variant_nh(int kv) { return kv == KV_WIDE ? kWideNH * kWidePPL : kTeamNH * kTeamPPL; }
// taps of the union of two adjacent columns' windows: x1(j+1) - x0(j) < s + 4*fs + 1
__host__ __device__ __forceinline__ int pair_union_bound(int in, int out) {
  const double s = (double)in / (double)out;
  const double fs = s > 1.0 ? s : 1.0;
  return (int)floor(s + 4.0 * fs + 1.0 + 1e-9);
}

// KV_GENERIC, or KV_DIRECT when a window exceeds the generic kernel's weight tables (4*max(in/out,1) + 2 taps
// > kGenericMaxTaps): those clips take the direct f64 kernel (vp_resize.cu), so every ratio is supported (C9).
__host__ __device__ __forceinline__ int generic_or_direct(int in_h, int in_w, int out_h, int out_w) {
  const double fv = (double)in_h / out_h, fh = (double)in_w / out_w;
  const double fs = fmax(fmax(fv, fh), 1.0);
  return 4.0 * fs + 2.0 > (double)kGenericMaxTaps ? KV_DIRECT : KV_GENERIC;
}

__host__ __device__ __forceinline__ int u8_rows_per_band(int in_h, int out_h) {
  const double s = (double)in_h / (double)out_h;
  return max(1, kU8Rows / (int)ceil(fmax(s, 1.0) / 4.0));
}
__host__ __device__ __forceinline__ int64_t u8_tiles(int n_frames, int in_h, int out_h, int out_w) {
  const int rb = u8_rows_per_band(in_h, out_h);
  return (int64_t)n_frames * ((out_h + rb - 1) / rb) * ((out_w + kU8Cols - 1) / kU8Cols);
}
// KV_U8 covers windows of <= kU8MaxTaps taps on both axes (downscales <= 15.5x); beyond: VP_EUNSUPPORTED
__host__ __device__ __forceinline__ bool u8_supported(int in_h, int in_w, int out_h, int out_w) {
  const double fs = fmax(fmax((double)in_h / out_h, (double)in_w / out_w), 1.0);
  return 4.0 * fs + 2.0 <= (double)kU8MaxTaps;
}

__host__ __device__ __forceinline__ int select_variant(int in_h, int in_w, int out_h, int out_w, int p,
                                                       int resize_mode = 0) {
  if (resize_mode == 1) return KV_U8;                    // VP_RESIZE_U8: the HF drop-in integer resize (N1)
  if (in_h == out_h && in_w == out_w && (p & 1) == 0) return KV_COPY;
  if (in_h >= out_h && in_w >= out_w && (p & 1) == 0 && in_h <= kTabInH && out_h <= kTabOutH &&
      pair_union_bound(in_w, out_w) <= kTeamUL) {
    if (in_w <= 128 * kWideNV && out_w <= 64 * kWideNH * kWidePPL && team_geometry(in_w, out_w, p, kWideNV, variant_nh(KV_WIDE)).ws > 0)
      return KV_WIDE;
    if (team_geometry(in_w, out_w, p, kTeamNV, variant_nh(KV_TEAM)).ws > 0) return KV_TEAM;
  }
  const double sv = (double)in_h / (double)out_h;
  // live output rows per source row <= floor(4/s)+1 for upscale (<= 5 iff s > 0.8) and <= 5 for downscale
  // (trimmed windows; brute-forced in tests/test_oracle_pixels.py::test_live_rows_bound).  The streaming kernel
  // stores column pairs (bf16x2 / float2), so it needs an even patch size.
  const double sh = (double)in_w / (double)out_w;
  if (!(p & 1) && sv > 0.8 && in_h <= kInHMax && out_h <= kOutHMax && sh >= 0.6 && fast_strip_width(in_w, out_w) >= 16) {
    const int th = axis_max_taps(in_w, out_w);
    for (int v = KV_MILD; v <= KV_STRONG; ++v)
      if (th <= fast_lhm(v)) return v;
  }
  // KV_TEAML (clips the fast streaming kernel cannot take, e.g. 1440p-4K sources at the Qwen budgets): the KV_TEAM
  // structure with column-pair windows up to kTeamULL taps; the 4-slot vertical ring holds for every downscale
  // (<= 4 live rows per source row)
  if (in_h >= out_h && in_w >= out_w && (p & 1) == 0 && in_h <= kTabInH && out_h <= kTabOutH &&
      pair_union_bound(in_w, out_w) <= kTeamULL && team_geometry(in_w, out_w, p, kTeamNV, variant_nh(KV_TEAM)).ws > 0)
    return KV_TEAML;
  return generic_or_direct(in_h, in_w, out_h, out_w);
}

}  // namespace vp
