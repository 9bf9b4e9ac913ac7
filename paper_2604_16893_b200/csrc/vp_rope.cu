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
// 4096-token chunks (8 consecutive tokens per thread), two block scans per chunk, carries between chunks.
#include "vp_internal.cuh"

namespace vp {
namespace {

constexpr int kRopeThreads = 512;
constexpr int kWarps = kRopeThreads / 32;
constexpr int kPer = 8;           // tokens per thread in the fill kernel

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
                                              int tps, int vlo, int vhi) {
  GridInfo r{};
  r.valid = false;
  r.iv = 1;
  if (typ == 1) {
    if (o >= n_images) return r;
    r.t = igrid[3 * o]; r.hh = igrid[3 * o + 1] / m; r.ww = igrid[3 * o + 2] / m;
  } else {
    if (o >= vcum[n_videos]) return r;
    int64_t v = o;
    if (variant == VP_ROPE_QWEN3_SPLIT) {       // last v with vcum[v] <= o, searched in [vlo, vhi]
      int lo = vlo, hi = vhi;
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

__global__ void __launch_bounds__(kRopeThreads, 2)
rope_fill_kernel(const int8_t* __restrict__ tt, const int64_t* __restrict__ cu, int B, int variant, int m,
                 const int64_t* __restrict__ igrid, int n_images, const int64_t* __restrict__ vgrid, int n_videos,
                 const double* __restrict__ spg, int tps, const int64_t* __restrict__ counts,
                 const int64_t* __restrict__ vcum, int64_t* __restrict__ pos, int64_t total_L,
                 int64_t* __restrict__ deltas, int32_t* __restrict__ status) {
  __shared__ int64_t sh2[kWarps][2];
  __shared__ int64_t shm[kWarps];
  __shared__ int s_bad, s_vlo, s_vhi;
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
  if (tid == 0) {
    s_bad = 0;
    // videos this sequence's runs can map to (QWEN3_SPLIT): those holding ordinals [bv, bv + its runs)
    int lo = 0, hi = n_videos > 0 ? n_videos - 1 : 0;
    if (variant == VP_ROPE_QWEN3_SPLIT && n_videos > 0) {
      auto find = [&](int64_t o) {
        int a = 0, z = n_videos - 1;
        while (a < z) {
          const int mid = (a + z + 1) >> 1;
          if (vcum[mid] <= o) a = mid; else z = mid - 1;
        }
        return a;
      };
      const int64_t nv = counts[2 * b + 1];
      lo = find(bv);
      hi = nv > 0 ? find(bv + nv - 1) : lo;
    }
    s_vlo = lo;
    s_vhi = hi;
  }
  __syncthreads();

  const int64_t s = cu[b], e = cu[b + 1], L = e - s;
  const int lane = tid & 31, warp = tid >> 5;
  int64_t c_text = 0, c_A = 0, c_ri = 0, c_rv = 0, c_start = 0;
  // Each thread owns kPer consecutive tokens of the chunk: three local passes (run starts; text count +
  // advances of the runs it starts; emit) around two block scans.  The grid of a run is looked up once
  // per run start (and once for a run continuing from the previous thread); the (t, h, w) offsets of a
  // visual token advance incrementally, so no per-token division or search remains.
  for (int64_t base = 0; base < L; base += (int64_t)kRopeThreads * kPer) {
    const int64_t k0 = base + (int64_t)tid * kPer;
    int ty[kPer];
    const int first_prev = (k0 > 0 && k0 < L) ? (int)tt[s + k0 - 1] : -1;   // -1: sequence start / idle
    int prevt = first_prev;
    int64_t ci = 0, cv = 0, lst = -1;
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int64_t k = k0 + u;
      ty[u] = k < L ? (int)tt[s + k] : -1;
      if (ty[u] >= 0 && ty[u] != prevt) {                   // run start (k == 0 always starts a run)
        if (ty[u] == 1) ++ci;
        else if (ty[u] == 2) ++cv;
        lst = k;
      }
      prevt = ty[u];
    }
    const int nextt = (k0 + kPer < L) ? (int)tt[s + k0 + kPer] : -1;
    int64_t x1[2] = {ci, cv}, t1[2];
    block_scan_sum<2>(x1, t1, sh2);
    const int64_t ri0 = c_ri + x1[0] - ci, rv0 = c_rv + x1[1] - cv;   // runs started before my first token
    // exclusive prefix max of the last run start (-> start of the run my first token continues)
    int64_t pm = lst;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, pm, o);
      if (lane >= o) pm = max(pm, y);
    }
    if (lane == 31) shm[warp] = pm;
    __syncthreads();
    int64_t before = __shfl_up_sync(0xffffffffu, pm, 1);
    if (lane == 0) before = -1;
    int64_t chunk_last = -1;
    for (int w = 0; w < kWarps; ++w) {
      if (w < warp) before = max(before, shm[w]);
      chunk_last = max(chunk_last, shm[w]);
    }
    __syncthreads();
    const int64_t rs0 = before >= 0 ? before : c_start;

    // pass 2: my text tokens and the advances A of the runs I start
    int64_t my_text = 0, my_A = 0;
    {
      int pt = first_prev;
      int64_t ri = ri0, rv = rv0;
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int typ = ty[u];
        if (typ == 0) ++my_text;
        else if (typ > 0 && typ != pt) {
          const int64_t o = typ == 1 ? bi + ri++ : bv + rv++;
          const GridInfo gi = grid_info(typ, o, variant, m, igrid, n_images, vgrid, n_videos, vcum, spg, tps, s_vlo, s_vhi);
          if (gi.valid) my_A += gi.A;
        }
        pt = typ;
      }
    }
    int64_t x2[2] = {my_text, my_A}, t2[2];
    block_scan_sum<2>(x2, t2, sh2);

    // pass 3: emit
    {
      int64_t tx = c_text + x2[0] - my_text, ax = c_A + x2[1] - my_A;
      int pt = first_prev;
      int64_t ri = ri0, rv = rv0, run_start = rs0, run_base = 0;
      GridInfo gi{};
      gi.valid = false;
      int64_t jt = 0, jh = 0, jw = 0;
      bool have = false;
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int typ = ty[u];
        const int64_t k = k0 + u, g = s + k;
        if (typ < 0) break;
        int64_t i0, i1, i2;
        if (typ == 0) {
          i0 = i1 = i2 = tx + ax;
          ++tx;
          have = false;
        } else {
          if (typ != pt) {                                   // run start
            const int64_t o = typ == 1 ? bi + ri++ : bv + rv++;
            gi = grid_info(typ, o, variant, m, igrid, n_images, vgrid, n_videos, vcum, spg, tps, s_vlo, s_vhi);
            run_start = k;
            run_base = tx + ax;
            if (gi.valid) ax += gi.A;
            jt = jh = jw = 0;
            have = true;
          } else if (!have) {                                // run continued from the previous thread
            const int64_t o = typ == 1 ? bi + ri - 1 : bv + rv - 1;
            gi = grid_info(typ, o, variant, m, igrid, n_images, vgrid, n_videos, vcum, spg, tps, s_vlo, s_vhi);
            run_base = tx + ax - (gi.valid ? gi.A : 0);
            const int64_t j = k - run_start;
            if (gi.valid && gi.tokens > 0) {
              const int64_t hw = gi.hh * gi.ww;
              jt = j / hw;
              jh = (j / gi.ww) % gi.hh;
              jw = j % gi.ww;
            }
            have = true;
          }
          if (gi.valid && gi.tokens > 0) {
            i0 = run_base + jt * gi.iv;
            i1 = run_base + jh;
            i2 = run_base + jw;
            if (++jw == gi.ww) { jw = 0; if (++jh == gi.hh) { jh = 0; ++jt; } }
          } else {
            i0 = i1 = i2 = run_base;
          }
          const int nt = u + 1 < kPer ? ty[u + 1] : nextt;
          if (nt != typ && (!gi.valid || (k - run_start + 1) != gi.tokens)) s_bad = 1;   // C24 strict check
        }
        pos[g] = i0;
        pos[total_L + g] = i1;
        pos[2 * total_L + g] = i2;
        pt = typ;
      }
    }
    c_text += t2[0];
    c_A += t2[1];
    c_ri += t1[0];
    c_rv += t1[1];
    if (chunk_last >= 0) c_start = chunk_last;
  }
  (void)block_max;
  __syncthreads();                                       // every thread's pass-3 s_bad write is visible to thread 0
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
