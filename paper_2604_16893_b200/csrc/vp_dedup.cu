// vp_dedup.cu -- N3: hash-based deduplication of the clips of a batch ("parallelizes
// [preprocessing] with hash-based deduplication"; GRPO draws n = 8 rollouts per prompt, so a rollout batch
// holds each clip n times).  The caller keys every sample's clip (e.g. a 64-bit hash of the video id and the
// sampling parameters); the library keeps the first occurrence of each key, the trainer plans and resizes only those
// clips, and every sample gets a view (patch offset + grid) into the unique clips' pixel_values.
//
//   dedup_kernel  (1 CTA): first[k] = smallest j <= k with keys[j] == keys[k] (threads compare their key with all
//                 earlier keys, O(n^2 / 1024) per thread: 512 samples take ~0.1 us of compares per thread), then a
//                 block scan of the first-occurrence flags gives the dense unique id of every sample and the list
//                 of unique samples in batch order.
//   views_kernel  per sample: its unique clip's patch offset and (t, h, w) from the unique clips' plans.
#include "vp_internal.cuh"

namespace vp {
namespace {

constexpr int kDedupThreads = 1024;

__global__ void __launch_bounds__(kDedupThreads)
dedup_kernel(const uint64_t* __restrict__ keys, int n, int32_t* __restrict__ unique_id,
             int32_t* __restrict__ unique_list, int32_t* __restrict__ n_unique) {
  __shared__ int wsum[kDedupThreads / 32];
  __shared__ int carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) carry = 0;
  __syncthreads();
  // pass 1: first occurrence of every key; dense ids of the first occurrences (block scan, batch order)
  for (int base = 0; base < n; base += kDedupThreads) {
    const int k = base + tid;
    int first = k;
    if (k < n) {
      const uint64_t key = keys[k];
      for (int j = 0; j < k; ++j)
        if (keys[j] == key) { first = j; break; }
    }
    const int flag = (k < n && first == k) ? 1 : 0;
    int x = flag;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    int before = carry;
    for (int w = 0; w < warp; ++w) before += wsum[w];
    const int id = before + x - flag;
    if (flag) {
      unique_id[k] = id;                  // first occurrences know their id now
      unique_list[id] = k;
    }
    __syncthreads();
    if (tid == kDedupThreads - 1) carry = before + x;
    __syncthreads();
  }
  if (tid == 0) *n_unique = carry;
  __syncthreads();
  // pass 2: repeats take the id of their first occurrence (written in pass 1; visible after the barriers)
  for (int k = tid; k < n; k += kDedupThreads) {
    const uint64_t key = keys[k];
    int first = k;
    for (int j = 0; j < k; ++j)
      if (keys[j] == key) { first = j; break; }
    if (first != k) unique_id[k] = unique_id[first];
  }
}

__global__ void views_kernel(const vp_clip_plan* __restrict__ uplans, const int32_t* __restrict__ unique_id, int n,
                             int64_t* __restrict__ patch_offset, int64_t* __restrict__ grid_thw,
                             int32_t* __restrict__ status) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const vp_clip_plan pl = uplans[unique_id[k]];
    const bool ok = pl.status == VP_OK;
    patch_offset[k] = ok ? pl.patch_offset : -1;
    grid_thw[3 * k + 0] = ok ? pl.grid_t : 0;
    grid_thw[3 * k + 1] = ok ? pl.grid_h : 0;
    grid_thw[3 * k + 2] = ok ? pl.grid_w : 0;
    if (status != nullptr) status[k] = pl.status;
  }
}

}  // namespace
}  // namespace vp

extern "C" vp_status vp_dedup_clips(const uint64_t* keys, int32_t n, int32_t* unique_id, int32_t* unique_list,
                                    int32_t* n_unique, void* stream) {
  if (n < 0 || (n > 0 && (keys == nullptr || unique_id == nullptr || unique_list == nullptr)) || n_unique == nullptr) {
    vp::set_error("vp_dedup_clips: invalid arguments");
    return VP_EINVAL;
  }
  vp::dedup_kernel<<<1, vp::kDedupThreads, 0, vp::as_stream(stream)>>>(keys, n, unique_id, unique_list, n_unique);
  return vp::launch_status("vp_dedup_clips");
}

extern "C" vp_status vp_dedup_views(const vp_clip_plan* unique_plans, const int32_t* unique_id, int32_t n,
                                    int64_t* patch_offset, int64_t* grid_thw, int32_t* status, void* stream) {
  if (n < 0 || (n > 0 && (unique_plans == nullptr || unique_id == nullptr || patch_offset == nullptr ||
                          grid_thw == nullptr))) {
    vp::set_error("vp_dedup_views: invalid arguments");
    return VP_EINVAL;
  }
  if (n == 0) return VP_OK;
  vp::views_kernel<<<(n + 255) / 256, 256, 0, vp::as_stream(stream)>>>(unique_plans, unique_id, n, patch_offset,
                                                                       grid_thw, status);
  return vp::launch_status("vp_dedup_views");
}
