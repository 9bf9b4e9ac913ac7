// vp_adjacent.cu -- N4: the steps adjacent to the hot path.
//   Upstream:   NV12 (the NVDEC output surface: Y plane + interleaved UV plane, 4:2:0) -> u8 RGB THWC frames in the
//               layout K3 reads (row pitch, frame stride), BT.601 limited range in the fixed-point form of OpenCV's
//               COLOR_YUV2RGB_NV12 (coefficients x 2^20, round by adding 2^19, arithmetic shift, saturate), so the
//               RGB bytes equal what a CPU decode stack hands the preprocessor.  P:73 "decodes, resamples, and
//               resizes"; codec decode itself is out of scope.
//   Downstream: the vision tower's per-patch 2D rotary position ids and the per-frame cu_seqlens of its
//               window-free attention (X: HF Qwen3-VL vision model rot_pos_emb / cu_seqlens), in pixel_values row
//               order (O8): row r of a (t, h, w) grid -> (hb*m + mh, wb*m + mw).
#include "vp_internal.cuh"
#include <algorithm>

namespace vp {
namespace {

constexpr int kCY = 1220542, kCUB = 2116026, kCUG = -409993, kCVG = -852492, kCVR = 1673527, kShift = 20;

__device__ __forceinline__ uint8_t sat8(int v) { return (uint8_t)(v < 0 ? 0 : (v > 255 ? 255 : v)); }

// One thread per 2x2 pixel block (one UV sample): reads 4 Y bytes + 2 UV bytes, writes 12 RGB bytes.
__global__ void nv12_kernel(const uint8_t* __restrict__ y, const uint8_t* __restrict__ uv, int64_t pitch,
                            int64_t frame_stride, int h, int w, int n_frames, uint8_t* __restrict__ out,
                            int64_t out_pitch, int64_t out_frame_stride) {
  const int bw = w >> 1, bh = h >> 1;
  const int64_t blocks = (int64_t)n_frames * bh * bw;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < blocks; e += (int64_t)gridDim.x * blockDim.x) {
    const int f = (int)(e / ((int64_t)bh * bw));
    const int rem = (int)(e - (int64_t)f * bh * bw);
    const int by = rem / bw, bx = rem - by * bw;
    const uint8_t* uvp = uv + (int64_t)f * frame_stride + (int64_t)by * pitch + 2 * bx;
    const int uu = (int)uvp[0] - 128, vv = (int)uvp[1] - 128;
    const int ruv = (1 << (kShift - 1)) + kCVR * vv;
    const int guv = (1 << (kShift - 1)) + kCVG * vv + kCUG * uu;
    const int buv = (1 << (kShift - 1)) + kCUB * uu;
#pragma unroll
    for (int dy = 0; dy < 2; ++dy) {
      const uint8_t* yp = y + (int64_t)f * frame_stride + (int64_t)(2 * by + dy) * pitch + 2 * bx;
      uint8_t* op = out + (int64_t)f * out_frame_stride + (int64_t)(2 * by + dy) * out_pitch + 6 * bx;
#pragma unroll
      for (int dx = 0; dx < 2; ++dx) {
        const int yy = max(0, (int)yp[dx] - 16) * kCY;
        op[3 * dx + 0] = sat8((yy + ruv) >> kShift);
        op[3 * dx + 1] = sat8((yy + guv) >> kShift);
        op[3 * dx + 2] = sat8((yy + buv) >> kShift);
      }
    }
  }
}

// Exclusive scans over the grids of patches (t*h*w) and frames (t), one CTA, chunks of 1024.
__global__ void __launch_bounds__(1024) vision_scan_kernel(const int64_t* __restrict__ grid, int n,
                                                           int64_t* __restrict__ patch_off,
                                                           int64_t* __restrict__ frame_off,
                                                           int32_t* __restrict__ cu_seqlens) {
  __shared__ int64_t wsum[32][2];
  __shared__ int64_t carry[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 2) carry[tid] = 0;
  __syncthreads();
  for (int base = 0; base < n; base += 1024) {
    const int k = base + tid;
    int64_t v[2] = {0, 0};
    if (k < n) {
      v[0] = grid[3 * k] * grid[3 * k + 1] * grid[3 * k + 2];
      v[1] = grid[3 * k];
    }
    int64_t x[2] = {v[0], v[1]};
#pragma unroll
    for (int j = 0; j < 2; ++j) {
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t t = __shfl_up_sync(0xffffffffu, x[j], o);
        if (lane >= o) x[j] += t;
      }
      if (lane == 31) wsum[warp][j] = x[j];
    }
    __syncthreads();
    int64_t before[2] = {carry[0], carry[1]};
    for (int w = 0; w < warp; ++w) { before[0] += wsum[w][0]; before[1] += wsum[w][1]; }
    if (k < n) {
      patch_off[k] = before[0] + x[0] - v[0];
      frame_off[k] = before[1] + x[1] - v[1];
    }
    __syncthreads();
    if (tid == 1023) { carry[0] = before[0] + x[0]; carry[1] = before[1] + x[1]; }
    __syncthreads();
  }
  if (tid == 0) { patch_off[n] = carry[0]; frame_off[n] = carry[1]; cu_seqlens[0] = 0; }
}

// Per grid (blockIdx.y strided): its patches' (row, col) ids and its frames' cu_seqlens entries.
__global__ void vision_fill_kernel(const int64_t* __restrict__ grid, int n, int m, const int64_t* __restrict__ patch_off,
                                   const int64_t* __restrict__ frame_off, int32_t* __restrict__ pos_ids,
                                   int32_t* __restrict__ cu_seqlens) {
  for (int g = blockIdx.y; g < n; g += gridDim.y) {
    const int64_t t = grid[3 * g], h = grid[3 * g + 1], w = grid[3 * g + 2];
    const int64_t hw = h * w, npatch = t * hw, p0 = patch_off[g];
    const int64_t wbn = w / m;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < npatch; r += (int64_t)gridDim.x * blockDim.x) {
      const int64_t s = r % hw;                       // patch within its frame (O8 order)
      const int64_t blk = s / (m * m), in = s - blk * (m * m);
      const int64_t hb = blk / wbn, wb = blk - hb * wbn, mh = in / m, mw = in - mh * m;
      pos_ids[2 * (p0 + r) + 0] = (int32_t)(hb * m + mh);
      pos_ids[2 * (p0 + r) + 1] = (int32_t)(wb * m + mw);
    }
    if (blockIdx.x == 0)
      for (int64_t f = threadIdx.x; f < t; f += blockDim.x) cu_seqlens[frame_off[g] + f + 1] = (int32_t)(p0 + (f + 1) * hw);
  }
}

}  // namespace
}  // namespace vp

extern "C" vp_status vp_nv12_to_rgb(const uint8_t* y, const uint8_t* uv, int64_t pitch, int64_t frame_stride,
                                    int32_t height, int32_t width, int32_t n_frames, uint8_t* rgb, int64_t rgb_pitch,
                                    int64_t rgb_frame_stride, void* stream) {
  if (height < 2 || width < 2 || (height & 1) || (width & 1) || n_frames < 0 || pitch < width ||
      rgb_pitch < 3 * (int64_t)width || (n_frames > 1 && (frame_stride < pitch * height ||
                                                          rgb_frame_stride < rgb_pitch * height)) ||
      (n_frames > 0 && (y == nullptr || uv == nullptr || rgb == nullptr))) {
    vp::set_error("vp_nv12_to_rgb: invalid arguments (even height/width >= 2, pitches, strides, pointers)");
    return VP_EINVAL;
  }
  if (n_frames == 0) return VP_OK;
  int dev = 0;
  cudaGetDevice(&dev);
  const int64_t blocks = (int64_t)n_frames * (height / 2) * (width / 2);
  const int grid = (int)std::min<int64_t>((blocks + 255) / 256, (int64_t)vp::device_sms(dev) * 8);
  vp::nv12_kernel<<<grid, 256, 0, vp::as_stream(stream)>>>(y, uv, pitch, frame_stride, height, width, n_frames, rgb,
                                                           rgb_pitch, rgb_frame_stride);
  return vp::launch_status("vp_nv12_to_rgb");
}

extern "C" size_t vp_vision_ids_workspace_bytes(int32_t n_grids) {
  return n_grids < 0 ? 0 : 2 * ((size_t)n_grids + 1) * sizeof(int64_t);
}

extern "C" vp_status vp_vision_ids(const int64_t* grid_thw, int32_t n_grids, int32_t merge_size, int32_t* pos_ids,
                                   int32_t* cu_seqlens, void* workspace, size_t workspace_bytes, void* stream) {
  if (n_grids < 0 || merge_size < 1 || (n_grids > 0 && (grid_thw == nullptr || pos_ids == nullptr)) ||
      cu_seqlens == nullptr || workspace == nullptr || workspace_bytes < vp_vision_ids_workspace_bytes(n_grids) ||
      (reinterpret_cast<uintptr_t>(workspace) & 7) != 0) {
    vp::set_error("vp_vision_ids: invalid arguments");
    return VP_EINVAL;
  }
  cudaStream_t s = vp::as_stream(stream);
  int64_t* po = reinterpret_cast<int64_t*>(workspace);
  int64_t* fo = po + n_grids + 1;
  vp::vision_scan_kernel<<<1, 1024, 0, s>>>(grid_thw, n_grids, po, fo, cu_seqlens);
  if (n_grids == 0) return vp::launch_status("vp_vision_ids");
  const dim3 g(8, (unsigned)std::min(n_grids, 65535));
  vp::vision_fill_kernel<<<g, 256, 0, s>>>(grid_thw, n_grids, merge_size, po, fo, pos_ids, cu_seqlens);
  return vp::launch_status("vp_vision_ids");
}
