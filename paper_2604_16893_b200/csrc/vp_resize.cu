// vp_resize.cu -- K2+K3: antialiased-bicubic resize -> clamp -> rescale/normalise -> temporal pad
// -> patchify, fused; every output element is written exactly once (O4-O9).
//
// This TU holds the dispatch (grids/status kernel, the fast variants of vp_resize_fast.cu, and the
// generic kernel) and the GENERIC kernel itself, which covers every ratio and alignment the fast
// variants do not (KV_GENERIC clips, and any clip whose frame buffer is not 16-B aligned).
//
// Generic work decomposition: persistent CTAs walk the token tiles of the clips they own, dealt
// round-robin.  A tile is (clip, temporal group g, merge-row band hb, merge-column strip wb): m*p x m*p
// output pixels of every frame slot of the group = m^2 consecutive pixel_values rows (one LLM token).
// Per tile, the AA weights of its m*p rows and m*p columns are computed in f64 and stored as fp32
// in shared memory (K2 as a prologue).  The separable filter then runs in two passes per source
// frame: vertical (u8 source rows -> fp32 rows of the column footprint, in shared memory) and
// horizontal (+ clamp + normalise + bf16/f32 store straight into the patch layout).
// A source frame that fills several temporal slots (odd n padding, images) is filtered once and
// stored to every slot.
#include "vp_k3_common.cuh"
#include <atomic>

namespace vp {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxTaps = kGenericMaxTaps;   // window length bound (~34x per axis); larger: KV_DIRECT
constexpr int kMaxBand = 64;           // m*p <= 64
constexpr int kVBufFloats = 8192;      // 32 KB vertical-pass buffer

struct KParams {
  int p, m, tp, D;                     // D = 3*tp*p*p
  float scale[3], bias[3];             // x = v*scale_c + bias_c = (v/255 - mean_c)/std_c
  int out_f32;
};

// Keys cubic (a = -0.5), f64 (C10)
__device__ __forceinline__ double keys(double x) {
  const double a = -0.5;
  x = fabs(x);
  if (x < 1.0) return ((a + 2.0) * x - (a + 3.0)) * x * x + 1.0;
  if (x < 2.0) return (((x - 5.0) * x + 8.0) * x - 4.0) * a;
  return 0.0;
}

// O4: AA window + normalised weights of output index i for an in->out axis.
// Returns window length (0 if it exceeds kMaxTaps: unsupported ratio).
__device__ int aa_window(int in, int out, int i, int* x0_out, float* w_out) {
  const double scale = (double)in / (double)out;
  const double fs = scale > 1.0 ? scale : 1.0;
  const double support = 2.0 * fs, inv = 1.0 / fs;
  const double c = ((double)i + 0.5) * scale;
  int x0 = (int)(c - support + 0.5);
  if (x0 < 0) x0 = 0;
  int x1 = (int)(c + support + 0.5);
  if (x1 > in) x1 = in;
  const int len = x1 - x0;
  if (len > kMaxTaps) return 0;
  double w[kMaxTaps];
  double s = 0.0;
  for (int k = 0; k < len; ++k) {
    w[k] = keys(((double)(k + x0) - c + 0.5) * inv);
    s += w[k];
  }
  const double r = s != 0.0 ? 1.0 / s : 1.0;
  for (int k = 0; k < len; ++k) w_out[k] = (float)(w[k] * r);
  *x0_out = x0;
  return len;
}

template <bool kF32>
__device__ __forceinline__ void store_px(void* base, int64_t idx, float x) {
  if (kF32) reinterpret_cast<float*>(base)[idx] = x;
  else reinterpret_cast<__nv_bfloat16*>(base)[idx] = __float2bfloat16_rn(x);
}

// ------------------------------------------------------------------------------------------
// Generic fused kernel (any ratio up to kMaxTaps-tap windows, any alignment).
// ------------------------------------------------------------------------------------------
template <bool kF32>
__global__ void __launch_bounds__(kThreads)
resize_generic_kernel(KParams kp, const vp_clip_plan* __restrict__ plans, int n, int fast_aligned,
                      const uint8_t* __restrict__ frames, const int64_t* __restrict__ clip_off,
                      const int64_t* __restrict__ pitch_arr, void* pv_img, int64_t img_cap, void* pv_vid,
                      int64_t vid_cap) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x;
  const int p = kp.p, m = kp.m, tp = kp.tp, B = m * p;
  float* s_v = reinterpret_cast<float*>(smem_raw);                 // [kVBufFloats]
  float* s_wv_base = s_v + kVBufFloats;                            // [B][kMaxTaps]
  float* s_wh_base = s_wv_base + B * kMaxTaps;                     // [B][kMaxTaps]
  int* s_vy0 = reinterpret_cast<int*>(s_wh_base + B * kMaxTaps);
  int* s_vlen = s_vy0 + B;
  int* s_hx0 = s_vlen + B;
  int* s_hlen = s_hx0 + B;
  int* s_bad_p = s_hlen + B;
#define s_wv(r) (s_wv_base + (r) * kMaxTaps)
#define s_wh(r) (s_wh_base + (r) * kMaxTaps)
#define s_bad (*s_bad_p)
  // Clips this kernel owns: KV_GENERIC, or fast-variant clips whose buffers are not 16-B aligned
  // (the fast kernel's TMA row copies need 16-B aligned rows).  Token tiles of every owned clip are
  // dealt round-robin over the CTAs, continuing the rotation across clips.
  // The plan list is scanned 256 clips at a time by the whole CTA (one clip per thread, block scan of
  // the owned tile counts), so a batch with no generic clip costs ~n/256 parallel steps, not n serial
  // plan loads per CTA.
  __shared__ int s_list[kThreads];
  __shared__ int64_t s_start[kThreads];
  __shared__ int64_t s_wsum[kThreads / 32];
  __shared__ int s_wcnt[kThreads / 32];
  int64_t rot = 0;
  for (int c0 = 0; c0 < n; c0 += kThreads) {
   const int kk = c0 + tid;
   int64_t my_tiles = 0;
   if (kk < n) {
     const vp_clip_plan& q = plans[kk];
     const bool fast_ok = fast_aligned && q.kernel_variant != KV_GENERIC && ((clip_off[kk] | pitch_arr[kk]) & 15) == 0;
     if (q.status == VP_OK && !fast_ok && q.kernel_variant != KV_DIRECT && q.kernel_variant != KV_U8)
       my_tiles = clip_tiles(q.grid_t, q.grid_h, q.grid_w, kp.m);
   }
   // block exclusive scan of (my_tiles, owned)
   const int lane = tid & 31, wid = tid >> 5;
   int64_t incl = my_tiles;
   int cnt = my_tiles > 0;
#pragma unroll
   for (int o = 1; o < 32; o <<= 1) {
     const int64_t a = __shfl_up_sync(0xffffffffu, incl, o);
     const int b = __shfl_up_sync(0xffffffffu, cnt, o);
     if (lane >= o) { incl += a; cnt += b; }
   }
   __syncthreads();                                  // previous chunk's s_list/s_start readers are done
   if (lane == 31) { s_wsum[wid] = incl; s_wcnt[wid] = cnt; }
   __syncthreads();
   int64_t wbase = 0, total = 0;
   int cbase = 0, ctotal = 0;
   for (int w = 0; w < kThreads / 32; ++w) {
     if (w < wid) { wbase += s_wsum[w]; cbase += s_wcnt[w]; }
     total += s_wsum[w]; ctotal += s_wcnt[w];
   }
   if (my_tiles > 0) {
     const int slot = cbase + cnt - 1;
     s_list[slot] = kk;
     s_start[slot] = rot + wbase + incl - my_tiles;
   }
   __syncthreads();
   for (int li = 0; li < ctotal; ++li) {
   const int k = s_list[li];
   const vp_clip_plan plk = plans[k];
   const int64_t ntile = clip_tiles(plk.grid_t, plk.grid_h, plk.grid_w, kp.m);
   const int64_t first = ((int64_t)blockIdx.x - s_start[li] % gridDim.x + gridDim.x) % gridDim.x;
   for (int64_t local = first; local < ntile; local += gridDim.x) {
    const vp_clip_plan& pl = plk;
    const int gh = pl.grid_h, gw = pl.grid_w;
    const int64_t tpg = (int64_t)(gh / m) * (gw / m);
    const int g = (int)(local / tpg);
    const int rem = (int)(local - (int64_t)g * tpg);
    const int hb = rem / (gw / m), wb = rem % (gw / m);
    void* pv = pl.is_image ? pv_img : pv_vid;
    const int64_t cap = pl.is_image ? img_cap : vid_cap;
    if (pv == nullptr || pl.patch_offset + (int64_t)pl.grid_t * gh * gw > cap) continue;  // ECAPACITY

    // ---- K2 prologue: AA weights for this tile's rows and columns (cached per clip for columns
    //      only when the strip repeats; recomputed per tile for simplicity) ----
    const int i0 = hb * B, j0 = wb * B;
    __syncthreads();
    if (tid == 0) s_bad = 0;
    __syncthreads();
    if (tid < B) {
      int x0, len = aa_window(pl.in_h, pl.out_h, i0 + tid, &x0, s_wv(tid));
      s_vy0[tid] = x0; s_vlen[tid] = len;
      if (len == 0) s_bad = 1;
    } else if (tid >= 128 && tid < 128 + B) {
      const int c = tid - 128;
      int x0, len = aa_window(pl.in_w, pl.out_w, j0 + c, &x0, s_wh(c));
      s_hx0[c] = x0; s_hlen[c] = len;
      if (len == 0) s_bad = 1;
    }
    __syncthreads();
    if (s_bad) continue;
    const int xa = s_hx0[0];
    const int xb = s_hx0[B - 1] + s_hlen[B - 1];
    const int fpb = 3 * (xb - xa);                 // footprint bytes per source row
    const int RS = min(B, kVBufFloats / fpb);       // output rows per sub-band
    if (RS < 1) continue;                           // unsupported (host checks the envelope)
    const int64_t pitch = pitch_arr[k];
    const int64_t frame_bytes = (int64_t)pl.in_h * pitch;
    const uint8_t* clip_base = frames + clip_off[k];
    const int64_t row_base = pl.patch_offset + (((int64_t)g * (gh / m) + hb) * (gw / m) + wb) * m * m;

    int ti = 0;
    while (ti < tp) {
      const int sf = min(g * tp + ti, pl.n_frames - 1);
      int ti_end = ti + 1;                           // slots [ti, ti_end) share source frame sf (O7)
      while (ti_end < tp && min(g * tp + ti_end, pl.n_frames - 1) == sf) ++ti_end;
      const uint8_t* src = clip_base + (int64_t)sf * frame_bytes + 3 * (int64_t)xa;

      for (int r0 = 0; r0 < B; r0 += RS) {
        const int nr = min(RS, B - r0);
        __syncthreads();
        // vertical pass: s_v[r][b] = sum_k wv[r0+r][k] * src[(y0+k)*pitch + b]
        for (int e = tid; e < nr * fpb; e += kThreads) {
          const int r = e / fpb, b = e - r * fpb;
          const int rr = r0 + r;
          const uint8_t* col = src + (int64_t)s_vy0[rr] * pitch + b;
          const int len = s_vlen[rr];
          float acc = 0.f;
          for (int kk = 0; kk < len; ++kk) acc = fmaf(s_wv(rr)[kk], (float)__ldg(col + (int64_t)kk * pitch), acc);
          s_v[r * fpb + b] = acc;
        }
        __syncthreads();
        // horizontal pass + clamp + normalise + store (consecutive threads -> consecutive px)
        for (int e = tid; e < nr * 3 * B; e += kThreads) {
          const int jj = e % B;
          const int rc = e / B;
          const int c = rc % 3, r = rc / 3;
          const float* vrow = s_v + r * fpb + 3 * (s_hx0[jj] - xa) + c;
          const int len = s_hlen[jj];
          float acc = 0.f;
          for (int l = 0; l < len; ++l) acc = fmaf(s_wh(jj)[l], vrow[3 * l], acc);
          acc = fminf(fmaxf(acc, 0.f), 255.f);                           // C12
          const float x = fmaf(acc, kp.scale[c], kp.bias[c]);             // O6
          const int il = r0 + r, mh = il / p, py = il - mh * p, mw = jj / p, px = jj - mw * p;
          const int64_t row = row_base + mh * m + mw;
          for (int t2 = ti; t2 < ti_end; ++t2) {
            const int64_t q = ((int64_t)(c * tp + t2) * p + py) * p + px;  // O8
            store_px<kF32>(pv, row * kp.D + q, x);
          }
        }
      }
      ti = ti_end;
    }
   }
   }
   rot += total;
  }
#undef s_wv
#undef s_wh
#undef s_bad
}

size_t generic_smem_bytes(int B) {
  return sizeof(float) * (kVBufFloats + 2 * (size_t)B * kMaxTaps) + sizeof(int) * (4 * B + 4);
}

// ------------------------------------------------------------------------------------------
// KV_DIRECT: downscales whose windows exceed the generic kernel's weight tables (> ~34x on an axis; rare:
// thumbnails of very large frames).  One thread per output pixel (all 3 channels) evaluates the separable
// AA-bicubic sum straight from the u8 source in f64 (O4-O6, C10-C13: the same window, Keys weights and
// renormalisation, no intermediate rounding), normalises, rounds once to the output dtype (O9) and stores into
// every temporal slot the frame fills (O7).  Work ~ (4s)^2 per output pixel, i.e. ~16x the source pixels.
// ------------------------------------------------------------------------------------------
struct Axis {
  int x0, x1;
  double c, inv, rsum;                 // window, centre, 1/fs, 1 / sum of its Keys weights
};
__device__ __forceinline__ Axis direct_axis(int in, int out, int i) {
  const double scale = (double)in / (double)out;
  const double fs = scale > 1.0 ? scale : 1.0;
  const double support = 2.0 * fs;
  Axis a;
  a.inv = 1.0 / fs;
  a.c = ((double)i + 0.5) * scale;
  a.x0 = max((int)(a.c - support + 0.5), 0);
  a.x1 = min((int)(a.c + support + 0.5), in);
  double s = 0.0;
  for (int x = a.x0; x < a.x1; ++x) s += keys(((double)x - a.c + 0.5) * a.inv);
  a.rsum = s != 0.0 ? 1.0 / s : 1.0;
  return a;
}

template <bool kF32>
__global__ void __launch_bounds__(256)
resize_direct_kernel(KParams kp, const vp_clip_plan* __restrict__ plans, int n, const uint8_t* __restrict__ frames,
                     const int64_t* __restrict__ clip_off, const int64_t* __restrict__ pitch_arr, void* pv_img,
                     int64_t img_cap, void* pv_vid, int64_t vid_cap, double mean0, double mean1, double mean2,
                     double std0, double std1, double std2) {
  const int p = kp.p, m = kp.m, tp = kp.tp, D = kp.D;
  const double mean[3] = {mean0, mean1, mean2}, sd[3] = {std0, std1, std2};
  for (int k = blockIdx.y; k < n; k += gridDim.y) {
    const vp_clip_plan pl = plans[k];
    if (pl.status != VP_OK || pl.kernel_variant != KV_DIRECT) continue;
    void* pv = pl.is_image ? pv_img : pv_vid;
    const int64_t cap = pl.is_image ? img_cap : vid_cap;
    if (pv == nullptr || pl.patch_offset + (int64_t)pl.grid_t * pl.grid_h * pl.grid_w > cap) continue;
    const int64_t pitch = pitch_arr[k];
    const int64_t hw = (int64_t)pl.out_h * pl.out_w;
    const int64_t npx = (int64_t)pl.n_frames * hw;
    const int gh = pl.grid_h / m, gw = pl.grid_w / m, B = m * p;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < npx; e += (int64_t)gridDim.x * blockDim.x) {
      const int f = (int)(e / hw);
      const int i = (int)((e - (int64_t)f * hw) / pl.out_w);
      const int j = (int)(e - (int64_t)f * hw - (int64_t)i * pl.out_w);
      const Axis av = direct_axis(pl.in_h, pl.out_h, i), ah = direct_axis(pl.in_w, pl.out_w, j);
      const uint8_t* src = frames + clip_off[k] + (int64_t)f * pl.in_h * pitch;
      double acc[3] = {0.0, 0.0, 0.0};
      for (int y = av.x0; y < av.x1; ++y) {
        const double wy = keys(((double)y - av.c + 0.5) * av.inv);
        if (wy == 0.0) continue;
        const uint8_t* row = src + (int64_t)y * pitch;
        double r[3] = {0.0, 0.0, 0.0};
        for (int x = ah.x0; x < ah.x1; ++x) {
          const double wx = keys(((double)x - ah.c + 0.5) * ah.inv);
          r[0] += wx * row[3 * x];
          r[1] += wx * row[3 * x + 1];
          r[2] += wx * row[3 * x + 2];
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) acc[c] += wy * r[c];
      }
      const int last = (f == pl.n_frames - 1) ? pl.grid_t * tp - 1 : f;   // frame n-1 fills the pad slots (O7)
      const int hb = i / B, mh = (i / p) % m, py = i % p, wb = j / B, mw = (j / p) % m, px = j % p;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double v = acc[c] * av.rsum * ah.rsum;
        v = v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v);                        // C12
        const float x = (float)((v / 255.0 - mean[c]) / sd[c]);              // O6 in f64, one rounding (O9)
        for (int sl = f; sl <= last; ++sl) {
          const int g = sl / tp, ti = sl - g * tp;
          const int64_t r = pl.patch_offset + (((int64_t)g * gh + hb) * gw + wb) * m * m + mh * m + mw;
          const int64_t q = ((int64_t)(c * tp + ti) * p + py) * p + px;
          if (kF32) reinterpret_cast<float*>(pv)[r * D + q] = x;
          else reinterpret_cast<__nv_bfloat16*>(pv)[r * D + q] = __double2bfloat16((v / 255.0 - mean[c]) / sd[c]);
        }
      }
    }
  }
}

// Grid outputs (H7) + per-clip status.  One small kernel; clips strided over threads.
__global__ void grids_kernel(const vp_clip_plan* __restrict__ plans, int n, int64_t img_cap, int64_t vid_cap,
                             int has_img, int has_vid, int64_t* __restrict__ img_grid, int64_t* __restrict__ vid_grid,
                             int32_t* __restrict__ clip_status) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const vp_clip_plan pl = plans[k];
    int32_t st = pl.status;
    if (st == VP_OK) {
      const int64_t rows = (int64_t)pl.grid_t * pl.grid_h * pl.grid_w;
      const bool img = pl.is_image;
      if (!(img ? has_img : has_vid) || pl.patch_offset + rows > (img ? img_cap : vid_cap)) st = VP_ECAPACITY;
      if (pl.kernel_variant == KV_U8 && !u8_supported(pl.in_h, pl.in_w, pl.out_h, pl.out_w)) st = VP_EUNSUPPORTED;
      int64_t* gptr = img ? img_grid : vid_grid;
      if (gptr != nullptr) {
        gptr[3 * pl.grid_index + 0] = pl.grid_t;
        gptr[3 * pl.grid_index + 1] = pl.grid_h;
        gptr[3 * pl.grid_index + 2] = pl.grid_w;
      }
    }
    if (clip_status != nullptr) clip_status[k] = st;
  }
}

constexpr int kMaxDev = 64;
std::atomic<unsigned> g_generic_attr[kMaxDev];

template <typename K>
void ensure_generic_attr(K kern, int dev, unsigned bit) {
  if (dev >= 0 && dev < kMaxDev && (g_generic_attr[dev].load(std::memory_order_acquire) & bit)) return;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (dev >= 0 && dev < kMaxDev) g_generic_attr[dev].fetch_or(bit, std::memory_order_acq_rel);
}

}  // namespace
}  // namespace vp

extern "C" size_t vp_resize_workspace_bytes(int32_t n) {
  return n < 0 ? 0 : vp::resize_ws_layout(n, nullptr).bytes;
}

extern "C" vp_status vp_resize_normalize_patchify(const vp_params* p, const vp_clip_plan* plans, int32_t n,
                                                  const uint8_t* frames,
                                                  const int64_t* clip_byte_offset, const int64_t* row_pitch,
                                                  void* pixel_values_images, int64_t img_rows_cap,
                                                  void* pixel_values_videos, int64_t vid_rows_cap,
                                                  int64_t* image_grid_thw, int64_t* video_grid_thw,
                                                  int32_t* clip_status, void* workspace, size_t workspace_bytes,
                                                  void* stream) {
  vp_status st = vp::check_params(p);
  if (st != VP_OK) return st;
  if (n < 0 || img_rows_cap < 0 || vid_rows_cap < 0) {
    vp::set_error("vp_resize_normalize_patchify: negative size argument");
    return VP_EINVAL;
  }
  if (n == 0) return VP_OK;
  if (plans == nullptr || frames == nullptr || clip_byte_offset == nullptr ||
      row_pitch == nullptr) {
    vp::set_error("vp_resize_normalize_patchify: null pointer argument");
    return VP_EINVAL;
  }
  const vp::ResizeWs ws = vp::resize_ws_layout(n, workspace);
  if (workspace == nullptr || workspace_bytes < ws.bytes || (reinterpret_cast<uintptr_t>(workspace) & 255) != 0) {
    vp::set_error("vp_resize_normalize_patchify: workspace must be >= vp_resize_workspace_bytes(%d) = %zu bytes, "
                  "256-B aligned (got %zu at %p)", n, ws.bytes, workspace_bytes, workspace);
    return VP_EINVAL;
  }
  if (p->merge_size * p->patch_size > vp::kMaxBand) {
    vp::set_error("vp_resize_normalize_patchify: merge_size*patch_size=%d exceeds %d",
                  p->merge_size * p->patch_size, vp::kMaxBand);
    return VP_EUNSUPPORTED;
  }
  cudaStream_t s = vp::as_stream(stream);
  int dev = 0;
  cudaGetDevice(&dev);
  const int sms = vp::device_sms(dev);
  vp::KParams kp{};
  kp.p = p->patch_size;
  kp.m = p->merge_size;
  kp.tp = p->temporal_patch_size;
  kp.D = 3 * kp.tp * kp.p * kp.p;
  for (int c = 0; c < 3; ++c) {
    kp.scale[c] = (float)(1.0 / (255.0 * p->std[c]));
    kp.bias[c] = (float)(-p->mean[c] / p->std[c]);
  }
  kp.out_f32 = p->out_dtype == VP_OUT_F32;
  vp::grids_kernel<<<(n + 255) / 256, 256, 0, s>>>(plans, n, img_rows_cap, vid_rows_cap,
                                                   pixel_values_images != nullptr, pixel_values_videos != nullptr,
                                                   image_grid_thw, video_grid_thw, clip_status);
  // launch hint (totals[VP_TOT_VARIANTS] of the plan): kernels of absent variants are not launched
  const unsigned mask = p->launch_mask != 0 ? (unsigned)p->launch_mask : ~0u;
  auto has = [&](int kv) { return (mask >> kv) & 1u; };
  const int fast_aligned = (reinterpret_cast<uintptr_t>(frames) & 15) == 0;
  const bool any_fast = has(vp::KV_MILD) || has(vp::KV_MEDIUM) || has(vp::KV_STRONG) || has(vp::KV_COPY) ||
                        has(vp::KV_TEAM) || has(vp::KV_WIDE) || has(vp::KV_TEAML);
  if ((fast_aligned && any_fast) || has(vp::KV_U8)) {
    const vp::FKParams fk = vp::make_fkparams(p);
    cudaError_t e = vp::launch_index(plans, n, clip_byte_offset, row_pitch, ws, sms, s);
    if (e == cudaSuccess && fast_aligned && (has(vp::KV_TEAM) || has(vp::KV_WIDE) || has(vp::KV_TEAML)))
      e = vp::launch_team(fk, plans, n, ws, frames, clip_byte_offset, row_pitch, pixel_values_images, img_rows_cap,
                          pixel_values_videos, vid_rows_cap, clip_status, dev, sms, mask, s);
    if (e == cudaSuccess && has(vp::KV_U8))
      e = vp::launch_u8(fk, plans, n, ws, frames, clip_byte_offset, row_pitch, pixel_values_images, img_rows_cap,
                        pixel_values_videos, vid_rows_cap, sms, s);
    if (e == cudaSuccess && fast_aligned)
      e = vp::launch_fast_variants(fk, plans, n, ws, frames, clip_byte_offset, row_pitch, pixel_values_images,
                                   img_rows_cap, pixel_values_videos, vid_rows_cap, dev, sms, mask, s);
    if (e != cudaSuccess) {
      vp::set_error("vp_resize_normalize_patchify: %s", cudaGetErrorString(e));
      return VP_ECUDA;
    }
  }
  if (has(vp::KV_DIRECT)) {
    const dim3 dg(16, (unsigned)(n < 65535 ? n : 65535));
    if (kp.out_f32)
      vp::resize_direct_kernel<true><<<dg, 256, 0, s>>>(kp, plans, n, frames, clip_byte_offset, row_pitch,
                                                        pixel_values_images, img_rows_cap, pixel_values_videos,
                                                        vid_rows_cap, p->mean[0], p->mean[1], p->mean[2], p->std[0],
                                                        p->std[1], p->std[2]);
    else
      vp::resize_direct_kernel<false><<<dg, 256, 0, s>>>(kp, plans, n, frames, clip_byte_offset, row_pitch,
                                                         pixel_values_images, img_rows_cap, pixel_values_videos,
                                                         vid_rows_cap, p->mean[0], p->mean[1], p->mean[2], p->std[0],
                                                         p->std[1], p->std[2]);
  }
  const int grid = sms * 3;
  const size_t smem = vp::generic_smem_bytes(kp.m * kp.p);
  if (kp.out_f32) {
    vp::ensure_generic_attr(vp::resize_generic_kernel<true>, dev, 1u);
    vp::resize_generic_kernel<true><<<grid, vp::kThreads, smem, s>>>(kp, plans, n, fast_aligned, frames, clip_byte_offset,
                                                                   row_pitch, pixel_values_images, img_rows_cap,
                                                                   pixel_values_videos, vid_rows_cap);
  } else {
    vp::ensure_generic_attr(vp::resize_generic_kernel<false>, dev, 2u);
    vp::resize_generic_kernel<false><<<grid, vp::kThreads, smem, s>>>(kp, plans, n, fast_aligned, frames, clip_byte_offset,
                                                                    row_pitch, pixel_values_images, img_rows_cap,
                                                                    pixel_values_videos, vid_rows_cap);
  }
  return vp::launch_status("vp_resize_normalize_patchify");
}
