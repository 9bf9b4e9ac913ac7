// vp_rope.cu -- K4: 3D MRoPE position ids + strict placeholder validation (O11).
//
// Position of token k of a sequence, as a scan (no sequential walk over runs):
//   p(k) = #text tokens before k + sum of A(run) over visual runs that started before k,
//   A(run) = max((t-1)*iv, h/m-1, w/m-1) + 1 (the run's advance; depends on its grid only).
// Text token: ids (p, p, p).  Visual token at offset j of run r (start s_r):
//   p_start = p(k) - (k > s_r ? A(r) : 0);  ids = p_start + (ti*iv, hi, wi), j -> (ti, hi, wi) row-major.
// The grid of a visual run is the o-th grid of its modality in batch order, o = run ordinal.
// Kernel A: per-sequence counts of visual runs (for batch-order ordinals) + video grid expansion
// prefix (QWEN3_SPLIT: video v contributes grid_t grids (1,h,w)).  Kernel B: one CTA per sequence,
// 512-token chunks, two block scans per chunk (warp shuffles), carries between chunks.
#include "vp_internal.cuh"

namespace vp {
namespace {

constexpr int kRopeThreads = 512;
constexpr int kWarps = kRopeThreads / 32;

// Inclusive block scan of NV int64 lanes (sum), returns inclusive values; totals in tot[].
template <int NV>
__device__ void block_scan_sum(int64_t (&x)[NV], int64_t (&tot)[NV], int64_t (*sh)[NV]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, x[j], o);
      if (lane >= o) x[j] += y;
    }
    if (lane == 31) sh[warp][j] = x[j];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      int64_t v = lane < kWarps ? sh[lane][j] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      if (lane < kWarps) sh[lane][j] = v;
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    if (warp > 0) x[j] += sh[warp - 1][j];
    tot[j] = sh[kWarps - 1][j];
  }
  __syncthreads();
}

__device__ __forceinline__ int64_t block_max(int64_t v, int64_t* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  int64_t r = sh[0];
  for (int w = 1; w < kWarps; ++w) r = max(r, sh[w]);
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(256)
rope_count_kernel(const int8_t* __restrict__ tt, const int64_t* __restrict__ cu, int B, int variant,
                  const int64_t* __restrict__ vgrid, int n_videos, int n_images, int64_t* __restrict__ counts,
                  int64_t* __restrict__ vcum, int32_t* __restrict__ status) {
  __shared__ int64_t sh[8][2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if ((int)blockIdx.x < B) {
    const int64_t s = cu[blockIdx.x], e = cu[blockIdx.x + 1];
    int64_t ci = 0, cv = 0;
    for (int64_t g = s + tid; g < e; g += blockDim.x) {
      const int8_t t = tt[g];
      if (t != 0 && (g == s || tt[g - 1] != t)) (t == 1 ? ci : cv) += 1;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ci += __shfl_xor_sync(0xffffffffu, ci, o);
      cv += __shfl_xor_sync(0xffffffffu, cv, o);
    }
    if (lane == 0) { sh[warp][0] = ci; sh[warp][1] = cv; }
    __syncthreads();
    if (tid == 0) {
      int64_t a = 0, b = 0;
      for (int w = 0; w < 8; ++w) { a += sh[w][0]; b += sh[w][1]; }
      counts[2 * blockIdx.x] = a;
      counts[2 * blockIdx.x + 1] = b;
    }
  } else {
    // exclusive prefix of grids contributed per video (split: grid_t, else 1); vcum[n_videos] = total
    __shared__ int64_t wsum[8];
    __shared__ int64_t carry;
    if (tid == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < n_videos; base += blockDim.x) {
      const int v = base + tid;
      int64_t c = v < n_videos ? (variant == VP_ROPE_QWEN3_SPLIT ? vgrid[3 * v] : 1) : 0;
      int64_t x = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) wsum[warp] = x;
      __syncthreads();
      int64_t pre = carry;
      for (int w = 0; w < warp; ++w) pre += wsum[w];
      if (v < n_videos) vcum[v] = pre + x - c;
      __syncthreads();
      if (tid == blockDim.x - 1) carry = pre + x;
      __syncthreads();
    }
    if (tid == 0) {
      vcum[n_videos] = carry;
      if (B == 0) status[0] = (n_images == 0 && carry == 0) ? VP_OK : VP_EMISMATCH;   // no sequences
    }
  }
}

struct GridInfo {
  int64_t t, hh, ww, iv, A, tokens;
  bool valid;
};

__device__ __forceinline__ GridInfo grid_info(int typ, int64_t o, int variant, int m, const int64_t* __restrict__ igrid,
                                              int n_images, const int64_t* __restrict__ vgrid, int n_videos,
                                              const int64_t* __restrict__ vcum, const double* __restrict__ spg,
                                              int tps) {
  GridInfo r{};
  r.valid = false;
  r.iv = 1;
  if (typ == 1) {
    if (o >= n_images) return r;
    r.t = igrid[3 * o]; r.hh = igrid[3 * o + 1] / m; r.ww = igrid[3 * o + 2] / m;
  } else {
    if (o >= vcum[n_videos]) return r;
    int64_t v = o;
    if (variant == VP_ROPE_QWEN3_SPLIT) {       // last v with vcum[v] <= o
      int lo = 0, hi = n_videos - 1;
      while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (vcum[mid] <= o) lo = mid; else hi = mid - 1;
      }
      v = lo;
      r.t = 1;
    } else {
      r.t = vgrid[3 * v];
    }
    r.hh = vgrid[3 * v + 1] / m; r.ww = vgrid[3 * v + 2] / m;
    if (variant == VP_ROPE_QWEN25) r.iv = (int64_t)tps * (int64_t)(spg != nullptr ? spg[v] : 1.0);
  }
  r.valid = true;
  r.tokens = r.t * r.hh * r.ww;
  r.A = max(max((r.t - 1) * r.iv, r.hh - 1), r.ww - 1) + 1;
  return r;
}

__global__ void __launch_bounds__(kRopeThreads)
rope_fill_kernel(const int8_t* __restrict__ tt, const int64_t* __restrict__ cu, int B, int variant, int m,
                 const int64_t* __restrict__ igrid, int n_images, const int64_t* __restrict__ vgrid, int n_videos,
                 const double* __restrict__ spg, int tps, const int64_t* __restrict__ counts,
                 const int64_t* __restrict__ vcum, int64_t* __restrict__ pos, int64_t total_L,
                 int64_t* __restrict__ deltas, int32_t* __restrict__ status) {
  __shared__ int64_t sh3[kWarps][3];
  __shared__ int64_t sh2[kWarps][2];
  __shared__ int64_t shm[kWarps];
  __shared__ int s_bad;
  const int b = blockIdx.x, tid = threadIdx.x;
  // batch-order base ordinals of this sequence's visual runs
  int64_t bi = 0, bv = 0, ai = 0, av = 0;
  for (int j = tid; j < B; j += kRopeThreads) {
    const int64_t ci = counts[2 * j], cv = counts[2 * j + 1];
    if (j < b) { bi += ci; bv += cv; }
    ai += ci; av += cv;
  }
  {
    int64_t x[4] = {bi, bv, ai, av}, tot[4];
    __shared__ int64_t sh4[kWarps][4];
    block_scan_sum<4>(x, tot, sh4);
    bi = tot[0]; bv = tot[1]; ai = tot[2]; av = tot[3];
  }
  if (b == 0 && tid == 0) {
    const int64_t n_vg = vcum[n_videos];
    status[B] = (ai == n_images && av == n_vg) ? VP_OK : VP_EMISMATCH;
  }
  if (tid == 0) s_bad = 0;
  __syncthreads();

  const int64_t s = cu[b], e = cu[b + 1], L = e - s;
  int64_t c_text = 0, c_A = 0, c_ri = 0, c_rv = 0, c_start = 0;
  for (int64_t base = 0; base < L; base += kRopeThreads) {
    const int64_t k = base + tid;
    const bool in = k < L;
    const int64_t g = s + k;
    const int typ = in ? tt[g] : 0;
    const bool start = in && (k == 0 || tt[g - 1] != typ);
    // scan 1: visual run starts per modality + run start position (max-scan)
    int64_t x1[2] = {start && typ == 1 ? 1 : 0, start && typ == 2 ? 1 : 0}, t1[2];
    block_scan_sum<2>(x1, t1, sh2);
    // run start: max over j <= k of (start_j ? j : -1), combined with the carry from earlier chunks
    int64_t st_pos = start ? k : -1;
    {
      // inclusive max-scan via warp shuffles + smem
      const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, st_pos, o);
        if (lane >= o) st_pos = max(st_pos, y);
      }
      if (lane == 31) shm[warp] = st_pos;
      __syncthreads();
      for (int w = 0; w < warp; ++w) st_pos = max(st_pos, shm[w]);
      __syncthreads();
    }
    const int64_t run_start = st_pos >= 0 ? st_pos : c_start;
    GridInfo gi{};
    gi.valid = false;
    gi.A = 0;
    int64_t o = -1;
    if (in && typ != 0) {
      const int64_t ord = (typ == 1 ? c_ri + x1[0] : c_rv + x1[1]) - 1;   // run ordinal within sequence
      o = (typ == 1 ? bi : bv) + ord;
      gi = grid_info(typ, o, variant, m, igrid, n_images, vgrid, n_videos, vcum, spg, tps);
    }
    // scan 2: text tokens and run advances (exclusive)
    const int64_t my_text = (in && typ == 0) ? 1 : 0;
    const int64_t my_A = (start && typ != 0 && gi.valid) ? gi.A : 0;
    int64_t x2[2] = {my_text, my_A}, t2[2];
    block_scan_sum<2>(x2, t2, sh2);
    const int64_t ex_text = x2[0] - my_text, ex_A = x2[1] - my_A;
    if (in) {
      int64_t p = c_text + ex_text + c_A + ex_A;
      int64_t i0, i1, i2;
      if (typ == 0) {
        i0 = i1 = i2 = p;
      } else {
        if (k > run_start && gi.valid) p -= gi.A;
        const int64_t j = k - run_start;
        if (gi.valid && gi.tokens > 0) {
          const int64_t hw = gi.hh * gi.ww;
          i0 = p + (j / hw) * gi.iv;
          i1 = p + (j / gi.ww) % gi.hh;
          i2 = p + j % gi.ww;
        } else {
          i0 = i1 = i2 = p;
        }
        const bool end = (k == L - 1) || tt[g + 1] != typ;
        if (end && (!gi.valid || (k - run_start + 1) != gi.tokens)) s_bad = 1;   // C24 strict check
      }
      pos[g] = i0;
      pos[total_L + g] = i1;
      pos[2 * total_L + g] = i2;
    }
    // carries
    c_text += t2[0];
    c_A += t2[1];
    c_ri += t1[0];
    c_rv += t1[1];
    {
      // run start of the chunk's last token
      __shared__ int64_t last_start;
      if (tid == kRopeThreads - 1) last_start = run_start;
      __syncthreads();
      c_start = last_start;
      __syncthreads();
    }
  }
  (void)block_max;
  if (tid == 0) {
    deltas[b] = L > 0 ? (c_text + c_A) - L : 0;        // max_id + 1 - len (C21)
    status[b] = s_bad ? VP_EMISMATCH : VP_OK;
  }
}

}  // namespace
}  // namespace vp

extern "C" size_t vp_rope_index_workspace_bytes(int32_t B, int32_t n_videos) {
  if (B < 0) B = 0;
  if (n_videos < 0) n_videos = 0;
  return ((size_t)2 * B + (size_t)n_videos + 1) * sizeof(int64_t) + 16;
}

extern "C" vp_status vp_rope_index(const vp_params* p, int32_t variant, const int8_t* mm_token_type,
                                   const int64_t* cu_seqlens, int32_t B, int64_t total_L,
                                   const int64_t* image_grid_thw, int32_t n_images,
                                   const int64_t* video_grid_thw, int32_t n_videos,
                                   const double* second_per_grid, int32_t tokens_per_second,
                                   int64_t* position_ids, int64_t* rope_deltas, int32_t* seq_status,
                                   void* workspace, size_t workspace_bytes, void* stream) {
  vp_status st = vp::check_params(p);
  if (st != VP_OK) return st;
  if (B < 0 || total_L < 0 || n_images < 0 || n_videos < 0 || variant < 0 || variant > 2) {
    vp::set_error("vp_rope_index: invalid sizes or variant (B=%d total_L=%lld variant=%d)", B, (long long)total_L,
                  variant);
    return VP_EINVAL;
  }
  if (cu_seqlens == nullptr || seq_status == nullptr || (B > 0 && rope_deltas == nullptr) ||
      (total_L > 0 && (mm_token_type == nullptr || position_ids == nullptr)) ||
      (n_images > 0 && image_grid_thw == nullptr) || (n_videos > 0 && video_grid_thw == nullptr) ||
      workspace == nullptr) {
    vp::set_error("vp_rope_index: null pointer argument");
    return VP_EINVAL;
  }
  if (workspace_bytes < vp_rope_index_workspace_bytes(B, n_videos) || (reinterpret_cast<uintptr_t>(workspace) & 15)) {
    vp::set_error("vp_rope_index: workspace too small or not 16-byte aligned (need %zu bytes)",
                  vp_rope_index_workspace_bytes(B, n_videos));
    return VP_EINVAL;
  }
  cudaStream_t s = vp::as_stream(stream);
  int64_t* counts = reinterpret_cast<int64_t*>(workspace);
  int64_t* vcum = counts + 2 * (size_t)B;
  vp::rope_count_kernel<<<B + 1, 256, 0, s>>>(mm_token_type, cu_seqlens, B, variant, video_grid_thw, n_videos,
                                              n_images, counts, vcum, seq_status);
  if (B > 0)  // B == 0: the count kernel writes the batch status
    vp::rope_fill_kernel<<<B, vp::kRopeThreads, 0, s>>>(mm_token_type, cu_seqlens, B, variant, p->merge_size,
                                                        image_grid_thw, n_images, video_grid_thw, n_videos,
                                                        second_per_grid, tokens_per_second, counts, vcum,
                                                        position_ids, total_L, rope_deltas, seq_status);
  return vp::launch_status("vp_rope_index");
}
