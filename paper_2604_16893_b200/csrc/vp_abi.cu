// vp_abi.cu -- host-side ABI plumbing: parameter validation, error text, status strings,
// struct-size probe, plus the two small H10 helpers (per-clip records for the all-gather and the
// global exclusive scan of the gathered records).
#include "vp_internal.cuh"
#include <cstdarg>
#include <cstring>

namespace vp {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

vp_status check_params(const vp_params* p) {
  if (p == nullptr) {
    set_error("params: null pointer");
    return VP_EINVAL;
  }
  const int64_t f = (int64_t)p->patch_size * p->merge_size;
  if (p->patch_size < 1 || p->merge_size < 1 || p->temporal_patch_size < 1) {
    set_error("params: patch_size, merge_size, temporal_patch_size must be >= 1");
    return VP_EINVAL;
  }
  if (p->max_frames < p->temporal_patch_size) {
    set_error("params: max_frames (%d) must be >= temporal_patch_size (%d) (S:33)", p->max_frames,
              p->temporal_patch_size);
    return VP_EINVAL;
  }
  if (p->video_max_pixels < f * f || p->image_max_pixels < f * f) {
    set_error("params: pixel budgets must be >= (patch*merge)^2 = %lld (S:32)", (long long)(f * f));
    return VP_EINVAL;
  }
  if (!(p->target_fps > 0.0) || p->min_pixels < 0 || (p->budget_mode != 0 && p->budget_mode != 1) ||
      (p->sampling != VP_SAMPLE_CENTER_BIN && p->sampling != VP_SAMPLE_LINSPACE) ||
      (p->out_dtype != 0 && p->out_dtype != 1) || p->min_frames < 0 || p->min_frames > p->max_frames ||
      (p->resize_mode != VP_RESIZE_FLOAT && p->resize_mode != VP_RESIZE_U8)) {
    set_error("params: invalid target_fps / min_pixels / budget_mode / sampling / out_dtype / min_frames / resize_mode");
    return VP_EINVAL;
  }
  for (int c = 0; c < 3; ++c)
    if (!(p->std[c] != 0.0)) {
      set_error("params: std[%d] must be non-zero", c);
      return VP_EINVAL;
    }
  return VP_OK;
}

vp_status launch_status(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: CUDA launch failed: %s", what, cudaGetErrorString(e));
    return VP_ECUDA;
  }
  return VP_OK;
}

namespace {
__global__ void records_kernel(const vp_clip_plan* __restrict__ plans, int n, int m, int32_t* __restrict__ rec) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const vp_clip_plan pl = plans[k];
    const bool ok = pl.status == VP_OK;
    rec[4 * k + 0] = ok ? pl.grid_t : 0;
    rec[4 * k + 1] = ok ? pl.grid_h : 0;
    rec[4 * k + 2] = ok ? pl.grid_w : 0;
    rec[4 * k + 3] = ok ? (int32_t)((int64_t)pl.grid_t * pl.grid_h * pl.grid_w / ((int64_t)m * m)) : 0;
  }
}

// Single CTA exclusive scan of tokens and patches over all gathered records (chunks of 1024).
__global__ void __launch_bounds__(1024) pack_kernel(const int32_t* __restrict__ rec, int total,
                                                    int64_t* __restrict__ tok, int64_t* __restrict__ pat) {
  __shared__ int64_t wsum[32][2];
  __shared__ int64_t carry[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 2) carry[tid] = 0;
  __syncthreads();
  for (int base = 0; base < total; base += 1024) {
    const int k = base + tid;
    int64_t v[2] = {0, 0};
    if (k < total) {
      v[0] = rec[4 * k + 3];
      v[1] = (int64_t)rec[4 * k] * rec[4 * k + 1] * rec[4 * k + 2];
    }
    int64_t x[2] = {v[0], v[1]};
#pragma unroll
    for (int j = 0; j < 2; ++j) {
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, x[j], o);
        if (lane >= o) x[j] += y;
      }
      if (lane == 31) wsum[warp][j] = x[j];
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        int64_t y0 = wsum[lane][j];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          int64_t y = __shfl_up_sync(0xffffffffu, y0, o);
          if (lane >= o) y0 += y;
        }
        wsum[lane][j] = y0;
      }
    }
    __syncthreads();
    int64_t ex[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) ex[j] = carry[j] + (warp ? wsum[warp - 1][j] : 0) + x[j] - v[j];
    if (k < total) {
      tok[k] = ex[0];
      pat[k] = ex[1];
    }
    __syncthreads();
    if (tid == 1023) {
      carry[0] = ex[0] + v[0];
      carry[1] = ex[1] + v[1];
    }
    __syncthreads();
  }
  if (tid == 0) {
    tok[total] = carry[0];
    pat[total] = carry[1];
  }
}
// N2 (Qwen2.5-VL time-scaled MRoPE): per video, second_per_grid_ts = temporal_patch_size / sampled_fps with HF's
// sampled fps n / total * src_fps (X: Qwen2_5_VLProcessor, VideoMetadata.sampled_fps), in that f64 order.
__global__ void spg_kernel(const vp_clip_desc* __restrict__ clips, const vp_clip_plan* __restrict__ plans, int n,
                           int tp, double* __restrict__ spg) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const vp_clip_plan pl = plans[k];
    if (pl.status != VP_OK || pl.is_image) continue;
    const double sampled = __dmul_rn(__ddiv_rn((double)pl.n_frames, (double)clips[k].total_source_frames),
                                     clips[k].source_fps);
    spg[pl.grid_index] = __ddiv_rn((double)tp, sampled);
  }
}
}  // namespace
}  // namespace vp

extern "C" {

vp_status vp_plan_second_per_grid(const vp_clip_desc* clips, const vp_clip_plan* plans, int32_t n,
                                  int32_t temporal_patch_size, double* second_per_grid, void* stream) {
  if (n < 0 || temporal_patch_size < 1 || (n > 0 && (clips == nullptr || plans == nullptr ||
                                                      second_per_grid == nullptr))) {
    vp::set_error("vp_plan_second_per_grid: invalid arguments");
    return VP_EINVAL;
  }
  if (n == 0) return VP_OK;
  vp::spg_kernel<<<(n + 255) / 256, 256, 0, vp::as_stream(stream)>>>(clips, plans, n, temporal_patch_size,
                                                                     second_per_grid);
  return vp::launch_status("vp_plan_second_per_grid");
}

const char* vp_status_string(vp_status s) {
  switch (s) {
    case VP_OK: return "VP_OK";
    case VP_EINVAL: return "VP_EINVAL: invalid argument";
    case VP_EALIGN: return "VP_EALIGN: misaligned pointer or pitch";
    case VP_EMISMATCH: return "VP_EMISMATCH: placeholder/feature count mismatch";
    case VP_ECAPACITY: return "VP_ECAPACITY: output buffer too small";
    case VP_ECUDA: return "VP_ECUDA: CUDA error";
    case VP_EUNSUPPORTED: return "VP_EUNSUPPORTED: unsupported size or ratio";
  }
  return "unknown vp_status";
}

const char* vp_last_error_detail(void) { return vp::g_err; }

int32_t vp_abi_version(void) { return VP_ABI_VERSION; }

int32_t vp_struct_sizes(void) {
  return (int32_t)(sizeof(vp_params) | (sizeof(vp_clip_desc) << 10) | (sizeof(vp_clip_plan) << 20));
}

vp_status vp_plan_records(const vp_clip_plan* plans, int32_t n, int32_t merge_size, int32_t* records, void* stream) {
  if (n < 0 || merge_size < 1 || (n > 0 && (plans == nullptr || records == nullptr))) {
    vp::set_error("vp_plan_records: invalid arguments");
    return VP_EINVAL;
  }
  if (n == 0) return VP_OK;
  vp::records_kernel<<<(n + 255) / 256, 256, 0, vp::as_stream(stream)>>>(plans, n, merge_size, records);
  return vp::launch_status("vp_plan_records");
}

vp_status vp_pack_offsets(const int32_t* gathered, int32_t world, int32_t clips_per_rank, int64_t* token_offsets,
                          int64_t* patch_offsets, void* stream) {
  if (world < 1 || clips_per_rank < 0 || gathered == nullptr || token_offsets == nullptr ||
      patch_offsets == nullptr) {
    vp::set_error("vp_pack_offsets: invalid arguments");
    return VP_EINVAL;
  }
  vp::pack_kernel<<<1, 1024, 0, vp::as_stream(stream)>>>(gathered, world * clips_per_rank, token_offsets,
                                                          patch_offsets);
  return vp::launch_status("vp_pack_offsets");
}

}  // extern "C"
