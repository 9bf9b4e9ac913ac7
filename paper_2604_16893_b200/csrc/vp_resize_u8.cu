// vp_resize_u8.cu -- N1 pixels: the HF drop-in resize (vp_params.resize_mode = VP_RESIZE_U8).  HF's processors
// resize uint8 frames on torch's uint8 antialiased-bicubic path; this kernel reproduces it bit for bit (pinned in
// the oracle against torch, tests/test_oracle_pixels.py) and then rescales + normalises (O6) and patchifies (O7-O9)
// like every other K3 kernel:
//   per axis, the C10 window and Keys weights (sequential f64 sum), quantised to int coefficients with precision
//   p = the largest p <= 22 with max|w| * 2^p < 2^15 over the axis, rounded half away from zero;
//   horizontal pass first: acc = 2^(p-1) + sum c_k x_k, out = clamp(acc >> p, 0, 255) as u8; then vertical.
// Work item (KV_U8, tile_count at plan time) = (clip, frame, band of RB output rows, strip of kU8Cols columns).
// Per CTA: the band's vertical and the strip's horizontal coefficients in shared memory, the horizontal pass of the
// tile's source rows into a u8 tile in shared memory, then the vertical pass, normalise and store straight into the
// patch layout.  Parity mode: not the bench path (each tile re-reads its halo).
#include "vp_k3_common.cuh"

namespace vp {
namespace {

__device__ __forceinline__ double keys_u8(double x) {
  const double a = -0.5;
  x = fabs(x);
  if (x < 1.0) return ((a + 2.0) * x - (a + 3.0)) * x * x + 1.0;
  if (x < 2.0) return (((x - 5.0) * x + 8.0) * x - 4.0) * a;
  return 0.0;
}

struct UWin {
  int x0, len;
  double c, inv, rsum;
};
// C10 window (untrimmed, as torch) with the sequential f64 weight sum
__device__ __forceinline__ UWin u8_window(int in, int out, int i) {
  const double s = (double)in / (double)out, fs = s > 1.0 ? s : 1.0, sup = 2.0 * fs;
  UWin w;
  w.inv = 1.0 / fs;
  w.c = ((double)i + 0.5) * s;
  w.x0 = max((int)(w.c - sup + 0.5), 0);
  w.len = min((int)(w.c + sup + 0.5), in) - w.x0;
  double t = 0.0;
  for (int k = 0; k < w.len; ++k) t += keys_u8(((double)(k + w.x0) - w.c + 0.5) * w.inv);
  w.rsum = t;
  return w;
}
__device__ __forceinline__ double u8_weight(const UWin& w, int k) {
  const double v = keys_u8(((double)(k + w.x0) - w.c + 0.5) * w.inv);
  return w.rsum != 0.0 ? v / w.rsum : v;
}
__device__ __forceinline__ int u8_coef(double w, int p) {
  const double v = w * (double)(1 << p);
  return v >= 0.0 ? (int)(v + 0.5) : (int)(v - 0.5);
}
// Per clip: the precision of each axis (max |w| over all its output indices).  One CTA per clip (strided).
__global__ void __launch_bounds__(256) u8_prec_kernel(const vp_clip_plan* __restrict__ plans, int n,
                                                      int2* __restrict__ prec) {
  __shared__ unsigned long long mx[2];
  for (int k = blockIdx.x; k < n; k += gridDim.x) {
    const vp_clip_plan pl = plans[k];
    if (pl.status != VP_OK || pl.kernel_variant != KV_U8) continue;
    if (threadIdx.x < 2) mx[threadIdx.x] = 0ull;
    __syncthreads();
    for (int a = 0; a < 2; ++a) {
      const int in = a ? pl.in_h : pl.in_w, out = a ? pl.out_h : pl.out_w;
      double m = 0.0;
      for (int i = threadIdx.x; i < out; i += blockDim.x) {
        const UWin w = u8_window(in, out, i);
        for (int t = 0; t < w.len; ++t) m = fmax(m, fabs(u8_weight(w, t)));
      }
      atomicMax(&mx[a], (unsigned long long)__double_as_longlong(m));   // non-negative: bit order = value order
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int pp[2];
      for (int a = 0; a < 2; ++a) {
        const double m = __longlong_as_double((long long)mx[a]);
        int p = 0;
        while (p < 22 && m * (double)(1 << (p + 1)) < 32768.0) ++p;
        pp[a] = p;
      }
      prec[k] = make_int2(pp[0], pp[1]);    // (horizontal, vertical)
    }
    __syncthreads();
  }
}

template <bool kF32>
__global__ void __launch_bounds__(256) resize_u8_kernel(FKParams kp, const vp_clip_plan* __restrict__ plans,
                                                        const VIdx vx, const int2* __restrict__ prec,
                                                        const uint8_t* __restrict__ frames,
                                                        const int64_t* __restrict__ clip_off,
                                                        const int64_t* __restrict__ pitch_arr, void* pv_img,
                                                        int64_t img_cap, void* pv_vid, int64_t vid_cap) {
  extern __shared__ __align__(16) unsigned char smem[];
  int* hc = reinterpret_cast<int*>(smem);                       // [kU8Cols][kU8MaxTaps] horizontal coefficients
  int* vc = hc + kU8Cols * kU8MaxTaps;                          // [kU8Rows][kU8MaxTaps] vertical coefficients
  int* hx0 = vc + kU8Rows * kU8MaxTaps;                         // [kU8Cols]
  int* hln = hx0 + kU8Cols;
  int* vy0 = hln + kU8Cols;                                     // [kU8Rows]
  int* vln = vy0 + kU8Rows;
  uint8_t* tile = reinterpret_cast<uint8_t*>(vln + kU8Rows);    // [rows][kU8Cols][3] horizontally resized u8
  const int cnt = (int)vx.meta[0];
  const int64_t total = vx.meta[1];
  const int p = kp.p, m = kp.m, tp = kp.tp, D = kp.D, B = m * p;
  for (int64_t item = blockIdx.x; item < total; item += gridDim.x) {
    const int j = vfind(vx, cnt, item);
    const int k = vx.list[j];
    const vp_clip_plan pl = plans[k];
    void* pv = pl.is_image ? pv_img : pv_vid;
    const int64_t cap = pl.is_image ? img_cap : vid_cap;
    if (pv == nullptr || pl.patch_offset + (int64_t)pl.grid_t * pl.grid_h * pl.grid_w > cap ||
        !u8_supported(pl.in_h, pl.in_w, pl.out_h, pl.out_w))
      continue;
    const int rb = u8_rows_per_band(pl.in_h, pl.out_h);
    const int nb = (pl.out_h + rb - 1) / rb, ns = (pl.out_w + kU8Cols - 1) / kU8Cols;
    const int64_t local = item - vx.off[j];
    const int f = (int)(local / ((int64_t)nb * ns));
    const int rem = (int)(local - (int64_t)f * nb * ns);
    const int b = rem / ns, st = rem - b * ns;
    const int i0 = b * rb, i1 = min(pl.out_h, i0 + rb), j0 = st * kU8Cols, j1 = min(pl.out_w, j0 + kU8Cols);
    const int2 pr = prec[k];
    __syncthreads();                                            // previous item's tile / tables are done
    // ---- coefficients of the strip's columns and the band's rows ----
    for (int q = threadIdx.x; q < (j1 - j0) + (i1 - i0); q += blockDim.x) {
      const bool col = q < j1 - j0;
      const int idx = col ? j0 + q : i0 + (q - (j1 - j0));
      const UWin w = col ? u8_window(pl.in_w, pl.out_w, idx) : u8_window(pl.in_h, pl.out_h, idx);
      int* c = col ? hc + q * kU8MaxTaps : vc + (q - (j1 - j0)) * kU8MaxTaps;
      const int len = min(w.len, kU8MaxTaps);
      for (int t = 0; t < len; ++t) c[t] = u8_coef(u8_weight(w, t), col ? pr.x : pr.y);
      if (col) { hx0[q] = w.x0; hln[q] = len; }
      else { vy0[q - (j1 - j0)] = w.x0; vln[q - (j1 - j0)] = len; }
    }
    __syncthreads();
    const int ys0 = vy0[0], ys1 = vy0[i1 - i0 - 1] + vln[i1 - i0 - 1];
    const int ncol = j1 - j0, nrow = ys1 - ys0;
    if (nrow > kU8TileRows) continue;                           // unreachable for supported ratios (<= 192 rows)
    const int64_t pitch = pitch_arr[k];
    const uint8_t* src = frames + clip_off[k] + (int64_t)f * pl.in_h * pitch;
    // ---- horizontal pass: source rows [ys0, ys1) -> u8 tile [nrow][ncol][3] ----
    const int hbias = 1 << (pr.x - 1);
    for (int e = threadIdx.x; e < nrow * ncol * 3; e += blockDim.x) {
      const int r = e / (ncol * 3), rem2 = e - r * ncol * 3, q = rem2 / 3, ch = rem2 - q * 3;
      const uint8_t* row = src + (int64_t)(ys0 + r) * pitch + ch;
      const int* c = hc + q * kU8MaxTaps;
      const int x0 = hx0[q], len = hln[q];
      int acc = hbias;
      for (int t = 0; t < len; ++t) acc += c[t] * (int)row[3 * (x0 + t)];
      acc >>= pr.x;
      tile[e] = (uint8_t)(acc < 0 ? 0 : (acc > 255 ? 255 : acc));
    }
    __syncthreads();
    // ---- vertical pass, normalise (O6), store into every temporal slot of frame f (O7, O8, O9) ----
    const int vbias = 1 << (pr.y - 1);
    const int last = (f == pl.n_frames - 1) ? pl.grid_t * tp - 1 : f;
    const int gh = pl.grid_h / m, gw = pl.grid_w / m;
    for (int e = threadIdx.x; e < (i1 - i0) * ncol * 3; e += blockDim.x) {
      const int r = e / (ncol * 3), rem2 = e - r * ncol * 3, q = rem2 / 3, ch = rem2 - q * 3;
      const int* c = vc + r * kU8MaxTaps;
      const int y0 = vy0[r] - ys0, len = vln[r];
      int acc = vbias;
      for (int t = 0; t < len; ++t) acc += c[t] * (int)tile[((y0 + t) * ncol + q) * 3 + ch];
      acc >>= pr.y;
      const float v = (float)(acc < 0 ? 0 : (acc > 255 ? 255 : acc));
      const float x = fmaf(v, kp.scale[ch], kp.bias[ch]);
      const int i = i0 + r, jj = j0 + q;
      const int hb = i / B, mh = (i / p) % m, py = i % p, wb = jj / B, mw = (jj / p) % m, px = jj % p;
      for (int sl = f; sl <= last; ++sl) {
        const int g = sl / tp, ti = sl - g * tp;
        const int64_t row = pl.patch_offset + (((int64_t)g * gh + hb) * gw + wb) * m * m + mh * m + mw;
        const int64_t col = ((int64_t)(ch * tp + ti) * p + py) * p + px;
        if (kF32) reinterpret_cast<float*>(pv)[row * D + col] = x;
        else reinterpret_cast<__nv_bfloat16*>(pv)[row * D + col] = __float2bfloat16_rn(x);
      }
    }
  }
}

}  // namespace

size_t u8_smem_bytes(int in_h_max_rows) {
  return sizeof(int) * ((size_t)(kU8Cols + kU8Rows) * kU8MaxTaps + 2 * kU8Cols + 2 * kU8Rows) +
         (size_t)in_h_max_rows * kU8Cols * 3;
}

cudaError_t launch_u8(const FKParams& kp, const vp_clip_plan* plans, int n, const ResizeWs& w, const uint8_t* frames,
                      const int64_t* coff, const int64_t* pitch, void* pi, int64_t icap, void* pvv, int64_t vcap,
                      int num_sms, cudaStream_t s) {
  u8_prec_kernel<<<min(n, 4 * num_sms), 256, 0, s>>>(plans, n, w.u8prec);
  const size_t smem = u8_smem_bytes(kU8TileRows);
  const VIdx vx = ws_vidx(w, n, 7);
  if (kp.out_f32) {
    cudaFuncSetAttribute(resize_u8_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    resize_u8_kernel<true><<<num_sms * 3, 256, smem, s>>>(kp, plans, vx, w.u8prec, frames, coff, pitch, pi, icap,
                                                          pvv, vcap);
  } else {
    cudaFuncSetAttribute(resize_u8_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    resize_u8_kernel<false><<<num_sms * 3, 256, smem, s>>>(kp, plans, vx, w.u8prec, frames, coff, pitch, pi, icap,
                                                           pvv, vcap);
  }
  return cudaGetLastError();
}

}  // namespace vp
