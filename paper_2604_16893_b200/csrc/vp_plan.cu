// vp_plan.cu -- K1: frame plan + smart_resize + grid + per-modality offsets + group timestamps.
//
// One CTA of 512 threads walks the clips in chunks of 512 (one thread per clip), does a
// block-wide exclusive scan (warp shuffles + one smem pass) of ten per-clip counters, and then
// writes frame indices / timestamps cooperatively (one warp per clip, lanes over frames).
// Planning is < 1 us of work even for thousands of clips; it is launch-latency bound by design.
//
// Bit-exactness (SURVEY §7 "hard parts"): every f64 expression uses explicit round-to-nearest
// intrinsics (__ddiv_rn/__dmul_rn/__dsqrt_rn/__dadd_rn) in the order the definition states,
// and this TU is compiled with --fmad=false, so the results equal IEEE evaluation on the host.
#include "vp_internal.cuh"

namespace vp {
namespace {

constexpr int kPlanThreads = 512;
constexpr int kNScan = 10;
enum { S_IDX = 0, S_IMGROWS, S_VIDROWS, S_IMGTOK, S_VIDTOK, S_NIMG, S_NVID, S_GROUPS, S_TILES, S_INVALID };

struct ClipResult {
  int32_t status, is_image, n, out_h, out_w, gt, gh, gw, variant;
  int64_t total;
  double src_fps, eff_fps;
};

// O2 smart_resize (readings C5-C8).  total_mode: area uses tb*hb*wb, scale term n*h*w.
__device__ void smart_resize(int64_t h, int64_t w, int64_t budget, int64_t f, int64_t min_px,
                             bool total_mode, int64_t n, int64_t tp, int32_t* H, int32_t* W) {
  int64_t hb = max(f, f * rne_div(h, f));
  int64_t wb = max(f, f * rne_div(w, f));
  int64_t area = hb * wb, term = h * w;
  if (total_mode) {
    area = ceil_div(n, tp) * tp * hb * wb;
    term = n * h * w;
  }
  if (area > budget) {
    double beta = __dsqrt_rn(__ddiv_rn((double)term, (double)budget));
    hb = max(f, (int64_t)floor(__ddiv_rn(__ddiv_rn((double)h, beta), (double)f)) * f);
    wb = max(f, (int64_t)floor(__ddiv_rn(__ddiv_rn((double)w, beta), (double)f)) * f);
  } else if (min_px > 0 && area < min_px) {
    double beta = __dsqrt_rn(__ddiv_rn((double)min_px, (double)term));
    hb = (int64_t)ceil(__ddiv_rn(__dmul_rn((double)h, beta), (double)f)) * f;
    wb = (int64_t)ceil(__ddiv_rn(__dmul_rn((double)w, beta), (double)f)) * f;
  }
  *H = (int32_t)hb;
  *W = (int32_t)wb;
}

__device__ ClipResult plan_one(const vp_params& P, const vp_clip_desc& c) {
  ClipResult r{};
  r.status = VP_EINVAL;
  r.is_image = c.is_image ? 1 : 0;
  const int64_t tp = P.temporal_patch_size, p = P.patch_size, m = P.merge_size, f = p * m;
  if (c.height < 1 || c.width < 1) return r;
  int64_t n;
  if (r.is_image) {
    n = 1;
    smart_resize(c.height, c.width, P.image_max_pixels, f, P.min_pixels, false, 1, tp, &r.out_h, &r.out_w);
  } else {
    // O1 (S:78 + C3): d = floor((total / src_fps) * target_fps)
    if (c.total_source_frames < 1 || !(c.source_fps > 0.0)) return r;
    double d = floor(__dmul_rn(__ddiv_rn((double)c.total_source_frames, c.source_fps), P.target_fps));
    if (P.sampling == VP_SAMPLE_LINSPACE) {
      // HF Qwen3-VL sample_frames: int(total / fps * target), min(max(n, min_frames), max_frames, total)
      if (d < (double)P.min_frames) n = P.min_frames;
      else if (d > (double)P.max_frames) n = P.max_frames;
      else n = (int64_t)d;
      n = min(n, (int64_t)P.max_frames);
      n = min(n, c.total_source_frames);
      if (n < 1) return r;
    } else {
      if (d < (double)tp) n = tp;
      else if (d > (double)P.max_frames) n = P.max_frames;
      else n = (int64_t)d;
      n = min(n, (int64_t)P.max_frames);
      n = min(n, c.total_source_frames);
      if (n >= tp) n = tp * (n / tp);
    }
    r.total = c.total_source_frames;
    r.src_fps = c.source_fps;
    // C23: effective fps = n*src_fps/total
    r.eff_fps = __ddiv_rn(__dmul_rn((double)n, c.source_fps), (double)c.total_source_frames);
    smart_resize(c.height, c.width, P.video_max_pixels, f, P.min_pixels, P.budget_mode == VP_BUDGET_TOTAL,
                 n, tp, &r.out_h, &r.out_w);
  }
  r.n = (int32_t)n;
  r.gt = (int32_t)ceil_div(n, tp);
  r.gh = r.out_h / (int32_t)p;
  r.gw = r.out_w / (int32_t)p;
  r.status = VP_OK;
  return r;
}

// HF linspace index: numpy linspace(0, total-1, n)[i] = i * ((total-1)/(n-1)) in f64 (last = total-1 exactly,
// n = 1 -> 0), rounded half to even (np.round).
__device__ __forceinline__ int64_t linspace_index(int64_t i, int64_t total, int64_t n) {
  if (n <= 1) return 0;
  if (i == n - 1) return total - 1;
  const double step = __ddiv_rn((double)(total - 1), (double)(n - 1));
  return (int64_t)rint(__dmul_rn((double)i, step));
}

// Center-of-bin index: min(total-1, floor((2i+1)*total / (2n))) in exact integers.
__device__ __forceinline__ int64_t frame_index(int64_t i, int64_t total, int64_t n) {
  const uint64_t a = (uint64_t)(2 * i + 1), t = (uint64_t)total;
  int64_t q;
  if (a <= (~0ull) / t) {                              // product fits 64 bits: plain u64 division
    q = (int64_t)((a * t) / (uint64_t)(2 * n));
  } else {
    unsigned __int128 num = (unsigned __int128)a * (unsigned __int128)t;
    q = (int64_t)(num / (unsigned __int128)(2 * n));
  }
  return q < total - 1 ? q : total - 1;
}

__device__ __forceinline__ int64_t sample_index(int sampling, int64_t i, int64_t total, int64_t n) {
  return sampling == VP_SAMPLE_LINSPACE ? linspace_index(i, total, n) : frame_index(i, total, n);
}

__global__ void __launch_bounds__(kPlanThreads, 1)
plan_kernel(vp_params P, const vp_clip_desc* __restrict__ clips, int n, vp_clip_plan* __restrict__ plans,
            int64_t* __restrict__ frame_indices, int64_t index_cap, double* __restrict__ ts, int64_t ts_cap,
            int64_t* __restrict__ totals) {
  __shared__ int64_t warp_tot[32][kNScan];
  __shared__ int64_t carry[kNScan];
  __shared__ int s_variants;                      // VP_TOT_VARIANTS: OR of 1 << kernel_variant over valid clips
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_variants = 0;
  const int64_t m2 = (int64_t)P.merge_size * P.merge_size;
  if (tid < kNScan) carry[tid] = 0;
  __syncthreads();

  for (int base = 0; base < n; base += kPlanThreads) {
    const int k = base + tid;
    ClipResult r{};
    r.status = VP_EINVAL;
    if (k < n) r = plan_one(P, clips[k]);
    const bool ok = (k < n) && r.status == VP_OK;
    int64_t patches = ok ? (int64_t)r.gt * r.gh * r.gw : 0;
    int64_t v[kNScan] = {0};
    if (ok) {
      v[S_IDX] = r.n;
      v[r.is_image ? S_IMGROWS : S_VIDROWS] = patches;
      v[r.is_image ? S_IMGTOK : S_VIDTOK] = patches / m2;
      v[r.is_image ? S_NIMG : S_NVID] = 1;
      v[S_GROUPS] = r.is_image ? 0 : r.gt;
      const int kv = select_variant(clips[k].height, clips[k].width, r.out_h, r.out_w, P.patch_size, P.resize_mode);
      r.variant = kv;
      atomicOr(&s_variants, 1 << kv);
      if (kv == KV_U8) {
        v[S_TILES] = u8_tiles(r.n, clips[k].height, r.out_h, r.out_w);
      } else if (kv == KV_COPY) {
        v[S_TILES] = (int64_t)r.n * (r.gh / P.merge_size) * copy_wchunks(r.gw, P.merge_size);
      } else if (kv == KV_TEAM || kv == KV_WIDE || kv == KV_TEAML) {
        v[S_TILES] = (int64_t)r.n *
                     team_geometry(clips[k].width, r.out_w, P.patch_size, variant_nv(kv), variant_nh(kv)).nslices;
      } else if (kv != KV_GENERIC) {
        const int ws = fast_strip_width(clips[k].width, r.out_w);
        v[S_TILES] = (int64_t)r.n * ((r.out_w + ws - 1) / ws);     // items: frames x strips
      }
    } else if (k < n) {
      v[S_INVALID] = 1;
    }
    // ---- block exclusive scan of v[] (H4) ----
    int64_t inc[kNScan];
#pragma unroll
    for (int j = 0; j < kNScan; ++j) {
      int64_t x = v[j];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      inc[j] = x;
      if (lane == 31) warp_tot[warp][j] = x;
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
      for (int j = 0; j < kNScan; ++j) {
        int64_t x = lane < kPlanThreads / 32 ? warp_tot[lane][j] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          int64_t y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        warp_tot[lane][j] = x;   // inclusive over warps
      }
    }
    __syncthreads();
    int64_t ex[kNScan];
#pragma unroll
    for (int j = 0; j < kNScan; ++j)
      ex[j] = carry[j] + (warp > 0 ? warp_tot[warp - 1][j] : 0) + inc[j] - v[j];
    if (k < n) {
      vp_clip_plan pl{};
      pl.status = r.status;
      pl.is_image = r.is_image;
      pl.in_h = clips[k].height;
      pl.in_w = clips[k].width;
      if (ok) {
        pl.n_frames = r.n;
        pl.out_h = r.out_h;
        pl.out_w = r.out_w;
        pl.grid_t = r.gt;
        pl.grid_h = r.gh;
        pl.grid_w = r.gw;
        pl.patch_offset = r.is_image ? ex[S_IMGROWS] : ex[S_VIDROWS];
        pl.token_offset = r.is_image ? ex[S_IMGTOK] : ex[S_VIDTOK];
        pl.grid_index = r.is_image ? ex[S_NIMG] : ex[S_NVID];
        pl.group_offset = r.is_image ? 0 : ex[S_GROUPS];
        pl.tile_count = (int32_t)v[S_TILES];
        pl.kernel_variant = r.variant;
        pl.effective_fps = r.eff_fps;
      }
      pl.index_offset = ex[S_IDX];
      pl.tile_offset = ex[S_TILES];   // monotone over all clips (invalid clips: count 0)
      plans[k] = pl;
    }
    __syncthreads();
    if (tid == kPlanThreads - 1) {
#pragma unroll
      for (int j = 0; j < kNScan; ++j) carry[j] = ex[j] + v[j];
    }
    __syncthreads();
  }
  if (tid == 0) {
    totals[VP_TOT_INDICES] = carry[S_IDX];
    totals[VP_TOT_IMG_ROWS] = carry[S_IMGROWS];
    totals[VP_TOT_VID_ROWS] = carry[S_VIDROWS];
    totals[VP_TOT_IMG_TOKENS] = carry[S_IMGTOK];
    totals[VP_TOT_VID_TOKENS] = carry[S_VIDTOK];
    totals[VP_TOT_N_IMAGES] = carry[S_NIMG];
    totals[VP_TOT_N_VIDEOS] = carry[S_NVID];
    totals[VP_TOT_VID_GROUPS] = carry[S_GROUPS];
    totals[VP_TOT_TILES] = carry[S_TILES];
    totals[VP_TOT_FLAGS] = 0;                     // plan_fill_kernel ORs overflow bits in
    totals[VP_TOT_N_INVALID] = carry[S_INVALID];
    totals[VP_TOT_VARIANTS] = s_variants;
  }
}


// ---- frame indices (O1) and group timestamps (O10): one warp per clip, many CTAs (the per-frame
//      integer divisions dominate K1 for long clips, so they are spread over the whole GPU) ----
constexpr int kFillThreads = 256;
__global__ void __launch_bounds__(kFillThreads)
plan_fill_kernel(int64_t tp, int sampling, const vp_clip_desc* __restrict__ clips, int n,
                 const vp_clip_plan* __restrict__ plans,
                 int64_t* __restrict__ frame_indices, int64_t index_cap, double* __restrict__ ts, int64_t ts_cap,
                 int64_t* __restrict__ totals) {
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * (kFillThreads / 32) + (threadIdx.x >> 5);
  if (c >= n) return;
  const vp_clip_plan& pl = plans[c];
  if (pl.status != VP_OK) return;
  unsigned long long flags = 0;
  const int64_t nn = pl.n_frames, off = pl.index_offset;
  if (pl.is_image) {
    if (lane == 0) {
      if (off < index_cap) frame_indices[off] = 0;
      else flags |= 1ull;
    }
  } else {
    const int64_t total = clips[c].total_source_frames;
    for (int64_t i = lane; i < nn; i += 32) {
      if (off + i < index_cap) frame_indices[off + i] = sample_index(sampling, i, total, nn);
      else flags |= 1ull;
    }
    if (ts != nullptr) {
      const double fps = clips[c].source_fps;
      const int64_t groups = ceil_div(nn, tp);
      for (int64_t g = lane; g < groups; g += 32) {
        int64_t i0 = g * tp, i1 = min(g * tp + tp - 1, nn - 1);   // pad with last index (C22)
        double a = __ddiv_rn((double)sample_index(sampling, i0, total, nn), fps);
        double b = __ddiv_rn((double)sample_index(sampling, i1, total, nn), fps);
        const int64_t o = pl.group_offset + g;
        if (o < ts_cap) ts[o] = __dmul_rn(__dadd_rn(a, b), 0.5);
        else flags |= 2ull;
      }
    }
  }
  flags = __reduce_or_sync(0xffffffffu, (unsigned)flags);
  if (lane == 0 && flags) atomicOr((unsigned long long*)&totals[VP_TOT_FLAGS], flags);
}

}  // namespace
}  // namespace vp

extern "C" vp_status vp_plan_frames(const vp_params* p, const vp_clip_desc* clips, int32_t n,
                                    vp_clip_plan* plans, int64_t* frame_indices, int64_t index_cap,
                                    double* group_timestamps, int64_t ts_cap, int64_t* totals, void* stream) {
  vp_status st = vp::check_params(p);
  if (st != VP_OK) return st;
  if (n < 0 || index_cap < 0 || ts_cap < 0) {
    vp::set_error("vp_plan_frames: n=%d index_cap=%lld ts_cap=%lld must be >= 0", n, (long long)index_cap,
                  (long long)ts_cap);
    return VP_EINVAL;
  }
  if (totals == nullptr || (n > 0 && (clips == nullptr || plans == nullptr)) ||
      (index_cap > 0 && frame_indices == nullptr)) {
    vp::set_error("vp_plan_frames: null pointer argument");
    return VP_EINVAL;
  }
  vp::plan_kernel<<<1, vp::kPlanThreads, 0, vp::as_stream(stream)>>>(*p, clips, n, plans, frame_indices,
                                                                      index_cap, group_timestamps, ts_cap, totals);
  if (n > 0) {
    const int per = vp::kFillThreads / 32;
    vp::plan_fill_kernel<<<(n + per - 1) / per, vp::kFillThreads, 0, vp::as_stream(stream)>>>(
        p->temporal_patch_size, p->sampling, clips, n, plans, frame_indices, index_cap, group_timestamps, ts_cap,
        totals);
  }
  return vp::launch_status("vp_plan_frames");
}
