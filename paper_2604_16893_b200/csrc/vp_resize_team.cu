// vp_resize_team.cu -- K3 "team" kernel: streaming fused AA-bicubic resize + clamp + normalise + temporal pad +
// patchify (O4-O9) for downscales / identity on both axes with a narrow horizontal window (KV_TEAM).
//
// Work item = (clip, slice, source frame f): a slice is a 16-column-aligned range of <= 64*kTeamW output columns
// whose source footprint fits kTeamW*128 pixels.  A CTA ("team") of kTeamW warps walks the item's source rows top
// to bottom exactly once.  Every warp does both passes (no producer/consumer warp specialisation):
//   V: the warp owns a 128-pixel (384-byte) part of the footprint; lane L converts its 12 bytes (4 RGB pixels) of
//      each staged source row once (I2F.U8 on the XU pipe for 2 of 3 words, PRMT + FADD2 for the third: both exact)
//      and FMAs them (FFMA2, broadcast weight) into a 4-slot register ring of live output rows.  For a downscale
//      (in >= out) at most 4 output rows are live at any source row (window 4s wide, centres s apart),
//      so 4 slots carry no dead FMAs at the bench ratio.  Output row i lives in slot i % 4; the output-row loop is
//      unrolled by 4 so every slot index -- and the parity of i, which picks the retire buffer -- is static.
//   retire: when output row i is complete, each lane stores its 4 pixels (float4 RGB + pad) into retire buffer
//      i & 1 (sub-pixel-major swizzle: conflict-free stores, ~1.3x wavefronts for the H taps), then ONE CTA barrier.
//   H: lane (warp w, lane l) owns output column pair q = 32w + l of the slice; the pair's union window (<= kUL taps,
//      weights (w_a, w_b) and swizzled tap offsets held in registers for the whole slice) is read once per row
//      (LDS.128) and FMA'd as 3 FFMA2 (pixel channel broadcast x pair weights); normalise (FFMA2), clamp in the
//      output domain, pack bf16x2 / float2 and store straight into the HF patch layout, once per temporal slot.
// Double-buffered retire rows + one barrier per output row are race-free: a warp writes buffer i&1 again only
// after passing barrier i+1, which every warp reaches after finishing its H of row i.
//
// Staging: each warp keeps kTDepth source rows of its part in flight with cp.async.bulk (refilled in groups of
// kTGrp rows, one mbarrier per group, producer state warp-uniform with the copies predicated to lane 0).  The
// vertical weights travel with the rows: per source row a 16-B record (the fp32 weights of its <= 4 live output
// rows, relative to the row being completed) copied by TMA from the per-clip table that team_vtab_kernel writes
// into the caller's workspace (f64 Keys / f64 window sum -> fp32, C10).  Consecutive clips of equal (in_h, out_h)
// share one table.
#include "vp_k3_common.cuh"
#include <atomic>

namespace vp {
namespace {

constexpr int kTW = kTeamW;                 // warps per CTA (team)
constexpr int kTT = kTW * 32;               // threads per CTA
#ifndef VP_TEAM_DEPTH
#define VP_TEAM_DEPTH 16
#endif
#ifndef VP_TEAM_PF
#define VP_TEAM_PF 0        // software-prefetch the next staged row (bytes + weight record) one row ahead
#endif
constexpr int kTDepth = VP_TEAM_DEPTH;      // staged source rows per warp
constexpr int kTGrp = 8;                    // rows per refill group (one mbarrier phase)
constexpr int kTNGrp = kTDepth / kTGrp;
constexpr int kTRowB = 400;                 // staged bytes per row slot: 384 + 16-B alignment slack
constexpr int kTPx = kTW * 128;             // footprint pixels per team (power of two)
static_assert((kTPx & (kTPx - 1)) == 0, "retire row index wraps with a mask");

struct TeamSmem {
  uint8_t stage[kTW][kTDepth][kTRowB];      // source rows
  float4 wrec[kTW][kTDepth];                // their vertical weight records
  float4 buf[2][kTPx];                      // retired output rows (swizzled pixel-major RGB + pad)
  uint64_t full[kTW][kTNGrp];               // staging groups: TMA -> warp
  int4 prod[kTW][3];                        // per-warp producer state (TeamProd)
};

// Per-warp producer state (warp-uniform; kept in shared memory between refills so that it does not occupy
// registers in the row loop).
struct TeamProd {
  const uint8_t* src;       // next source row of this warp's part (16-B aligned)
  const float4* wr;         // its weight record
  int64_t pitch;
  int64_t next;             // next item to open
  int rows, nbytes;         // rows left in the current item, bytes copied per row
};
static_assert(sizeof(TeamProd) <= 3 * sizeof(int4), "TeamProd");

// Slice geometry of an item: output columns [j0, j0+jn), footprint pixels [pa, pa+np) with pa a multiple of 4.
struct TItem {
  int j;                    // position in the variant list
  int k;                    // clip index
  int s, f;                 // slice, frame
};

__device__ __forceinline__ TItem decode_item(const VIdx& vx, int cnt, int64_t item, const vp_clip_plan* plans, int p,
                                             int* ws_out) {
  TItem t;
  t.j = vfind(vx, cnt, item);
  t.k = vx.list[t.j];
  const vp_clip_plan& pl = plans[t.k];
  const TeamGeo g = team_geometry(pl.in_w, pl.out_w, p);
  const int64_t local = item - vx.off[t.j];
  t.s = (int)(local / pl.n_frames);            // slice-major: consecutive items share the slice's H weights
  t.f = (int)(local - (int64_t)t.s * pl.n_frames);
  *ws_out = g.ws;
  return t;
}

__device__ __forceinline__ void slice_span(const vp_clip_plan& pl, int ws, int s, int& j0, int& jn, int& pa, int& np) {
  j0 = s * ws;
  jn = min(ws, pl.out_w - j0);
  pa = window_of(pl.in_w, pl.out_w, j0).x0 & ~3;
  np = window_of(pl.in_w, pl.out_w, j0 + jn - 1).x1 - pa;
}

__device__ __forceinline__ float2& h2(float4& v, int h) { return reinterpret_cast<float2*>(&v)[h]; }

// Retired-row swizzle (pixel-major float4 at vpos(x)): inside each 32-pixel block, sub-pixel-major (pixel 4a+k at
// 8k+a) -- the V lanes' stores (pixels 4L+k) hit 8 distinct 16-B granules per quarter-warp.
__device__ __forceinline__ int tpos(int x) {
  x &= kTPx - 1;
  return (x & ~31) | ((x & 3) << 3) | ((x & 31) >> 2);
}

// bytes -> floats: I2F.U8 (XU pipe) or PRMT into 2^23 + b then FADD2 -2^23 (ALU + FMA pipes); both exact.
__device__ __forceinline__ void cvt_i2f(uint32_t w, float2& lo, float2& hi) {
  lo = make_float2((float)(w & 0xffu), (float)((w >> 8) & 0xffu));
  hi = make_float2((float)((w >> 16) & 0xffu), (float)(w >> 24));
}
__device__ __forceinline__ void cvt_magic(uint32_t w, float2& lo, float2& hi) {
  const float2 mm = make_float2(-8388608.f, -8388608.f);
  lo = __fadd2_rn(make_float2(__uint_as_float(__byte_perm(w, 0x4B000000u, 0x7540u)),
                              __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7541u))), mm);
  hi = __fadd2_rn(make_float2(__uint_as_float(__byte_perm(w, 0x4B000000u, 0x7542u)),
                              __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7543u))), mm);
}

// One source row into the ring: output rows i..i+3 (i in slot U) get weights w.x..w.w.
template <int U>
__device__ __forceinline__ void ring4(float4 (&acc)[4][3], const float4 w, const float2 (&f)[6]) {
  const float ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int slot = (U + r) & 3;
    const float2 ww = make_float2(ws[r], ws[r]);
#pragma unroll
    for (int q = 0; q < 6; ++q) h2(acc[slot][q >> 1], q & 1) = __ffma2_rn(ww, f[q], h2(acc[slot][q >> 1], q & 1));
  }
}

// normalise (O6) as FFMA2 over the column pair, clamp (C12) in the output domain (clamp(v,0,255)*s+b ==
// clamp(v*s+b, lo, hi) with lo/hi the images of 0 and 255, ordered), round (O9) and store the pair into every
// temporal slot the frame fills (O7); for bf16 RNE is monotone, so clamping the rounded pair is bit-identical.
template <bool kF32>
__device__ __forceinline__ void store_pair(const FKParams& kp, char* q, float2 ar, float2 ag, float2 ab, int cstride,
                                           int nslots, int ti0, int tp, int p, int64_t group_stride) {
  constexpr int kEsz = kF32 ? 4 : 2;
  const float2 n[3] = {__ffma2_rn(ar, make_float2(kp.scale[0], kp.scale[0]), make_float2(kp.bias[0], kp.bias[0])),
                       __ffma2_rn(ag, make_float2(kp.scale[1], kp.scale[1]), make_float2(kp.bias[1], kp.bias[1])),
                       __ffma2_rn(ab, make_float2(kp.scale[2], kp.scale[2]), make_float2(kp.bias[2], kp.bias[2]))};
  uint2 o[3];                                      // per channel: the pair as float2 (f32) or bf16x2 in .x (bf16)
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    if (kF32) {
      const float2 v = make_float2(fminf(fmaxf(n[c].x, kp.lo[c]), kp.hi[c]), fminf(fmaxf(n[c].y, kp.lo[c]), kp.hi[c]));
      o[c] = make_uint2(__float_as_uint(v.x), __float_as_uint(v.y));
    } else {
      const __nv_bfloat162 v = __hmin2(__hmax2(__floats2bfloat162_rn(n[c].x, n[c].y), kp.lo2[c]), kp.hi2[c]);
      o[c].x = *reinterpret_cast<const uint32_t*>(&v);
    }
  }
  auto put = [&](char* d) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      if (kF32) *reinterpret_cast<uint2*>(d + (int64_t)c * cstride * kEsz) = o[c];
      else *reinterpret_cast<uint32_t*>(d + (int64_t)c * cstride * kEsz) = o[c].x;
    }
  };
  put(q);
  if (nslots > 1) {                                // frame n-1 also fills the temporal pad slots (O7)
    for (int s2 = 1, ti = ti0; s2 < nslots; ++s2) {
      if (++ti == tp) { ti = 0; q += (group_stride - (int64_t)(tp - 1) * p * p) * kEsz; } else q += (int64_t)p * p * kEsz;
      put(q);
    }
  }
}

#ifndef VP_TEAM_MINB
#define VP_TEAM_MINB 3      // CTAs per SM the register budget is sized for (3: 168 registers, no spills)
#endif
template <int kUL, bool kF32, int P, int M, int TP>
__global__ void __launch_bounds__(kTT, VP_TEAM_MINB)
resize_team_kernel(FKParams kp, const vp_clip_plan* __restrict__ plans, const VIdx vx, const int* __restrict__ tab_alias,
                   const int* __restrict__ tab_flag, const float4* __restrict__ vtab, const int* __restrict__ y1tab, const uint8_t* __restrict__ frames,
                   const int64_t* __restrict__ clip_off, const int64_t* __restrict__ pitch_arr, void* pv_img,
                   int64_t img_cap, void* pv_vid, int64_t vid_cap, int32_t* __restrict__ clip_status) {
  __shared__ __align__(128) TeamSmem sm;
  const int tid = threadIdx.x;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  int lane;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(lane));
  const bool l0 = lane == 0;

  const int cnt = (int)vx.meta[0];
  const int64_t total = vx.meta[1];
  const int64_t my_a = total * blockIdx.x / gridDim.x;
  const int64_t my_b = total * (blockIdx.x + 1) / gridDim.x;
  if (my_a >= my_b) return;

  if (tid == 0) {
    for (int w = 0; w < kTW; ++w)
      for (int g = 0; g < kTNGrp; ++g) mbar_init(&sm.full[w][g], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < 2 * kTPx; i += kTT) (&sm.buf[0][0])[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  __syncthreads();

  // ------------------------------------------------------------------ producer (this warp's part)
  uint8_t* stage = &sm.stage[warp][0][0];
  float4* wrec = &sm.wrec[warp][0];
  uint64_t* full = &sm.full[warp][0];
  TeamProd* ps = reinterpret_cast<TeamProd*>(&sm.prod[warp][0]);
  if (l0) {
    TeamProd z;
    z.src = nullptr; z.wr = nullptr; z.pitch = 0; z.next = my_a; z.rows = 0; z.nbytes = 0;
    *ps = z;
  }
  __syncwarp();
  auto open_item = [&](TeamProd& st) {          // warp-uniform
    int ws;
    const TItem t = decode_item(vx, cnt, st.next, plans, P > 0 ? P : kp.p, &ws);
    const vp_clip_plan& pl = plans[t.k];
    int j0, jn, pa, np;
    slice_span(pl, ws, t.s, j0, jn, pa, np);
    const int px0 = pa + warp * 128;
    const int pxn = min(128, np - warp * 128);
    const int b0 = 3 * px0;
    const int o = b0 & 15;
    st.nbytes = pxn > 0 ? ((o + 3 * pxn + 15) & ~15) : 0;
    st.pitch = pitch_arr[t.k];
    st.src = frames + clip_off[t.k] + (int64_t)t.f * pl.in_h * st.pitch + (b0 - o);
    st.wr = vtab + (int64_t)tab_alias[t.j] * kTabInH;
    st.rows = pl.in_h;
    ++st.next;
  };
  auto issue_group = [&](uint32_t g) {
    asm volatile("mov.b32 %0, %0;" : "+r"(g));   // opaque copy (nvcc 12.9 mbarrier-address CSE workaround)
    TeamProd st = *ps;
    if (st.rows >= kTGrp) {
      mbar_expect_tx_if(&full[g], (uint32_t)(kTGrp * st.nbytes + kTGrp * 16), l0);
#pragma unroll
      for (int q = 0; q < kTGrp; ++q)
        tma_bulk_g2s_if(stage + (size_t)(g * kTGrp + q) * kTRowB, st.src + (int64_t)q * st.pitch, (uint32_t)st.nbytes,
                        &full[g], l0 && st.nbytes > 0);
      tma_bulk_g2s_if(wrec + g * kTGrp, st.wr, kTGrp * 16, &full[g], l0);
      st.src += (int64_t)kTGrp * st.pitch;
      st.wr += kTGrp;
      st.rows -= kTGrp;
    } else {
#pragma unroll 1
      for (int q = 0; q < kTGrp; ++q) {
        if (st.rows == 0 && st.next < my_b) open_item(st);
        if (st.rows > 0) {
          mbar_expect_tx_if(&full[g], (uint32_t)(st.nbytes + 16), l0);
          tma_bulk_g2s_if(stage + (size_t)(g * kTGrp + q) * kTRowB, st.src, (uint32_t)st.nbytes, &full[g],
                          l0 && st.nbytes > 0);
          tma_bulk_g2s_if(wrec + g * kTGrp + q, st.wr, 16, &full[g], l0);
          st.src += st.pitch;
          st.wr += 1;
          --st.rows;
        }
      }
    }
    mbar_arrive_if(&full[g], l0);
    __syncwarp();
    if (l0) *ps = st;
    __syncwarp();
  };
  for (uint32_t g = 0; g < kTNGrp; ++g) issue_group(g);

  // ------------------------------------------------------------------ consumer
  // model geometry: compile-time for the preset instantiations (P > 0), runtime otherwise
  const int p = P > 0 ? P : kp.p, m = P > 0 ? M : kp.m, tp = P > 0 ? TP : kp.tp;
  const int B = m * p, D = 3 * tp * p * p;
  const int cstride = tp * p * p;                 // elements between channel blocks of a patch row (O8)
  constexpr int kEsz = kF32 ? 4 : 2;
  uint32_t rc = 0;                                // staged rows consumed: slot rc % kTDepth
  int cur_j = -1, cur_s = -1;
  // per-slice H state (registers): pair weights and swizzled tap shared addresses
  float2 wp[kUL];
  uint32_t toff[kUL];                             // shared addresses of the taps in retire buffer 0
  int colpart = 0;
  bool hact = false;
  const uint32_t buf_s = smem_u32(&sm.buf[0][0]);
  // V retire address of this lane's 4 pixels (pixel 128*warp + 4*lane + k at +128k)
  const uint32_t vsa = buf_s + (uint32_t)tpos(warp * 128 + lane * 4) * 16u;
  const uint32_t stage_s = smem_u32(stage), wrec_s = smem_u32(wrec);

  for (int64_t item = my_a; item < my_b; ++item) {
    int ws;
    const TItem t = decode_item(vx, cnt, item, plans, p, &ws);
    const vp_clip_plan& pl = plans[t.k];
    const int in_h = pl.in_h, out_h = pl.out_h;
    int j0, jn, pa, np;
    slice_span(pl, ws, t.s, j0, jn, pa, np);
    const int ta = tab_alias[t.j];
    const int* y1 = y1tab + (int64_t)ta * kTabOutH;
    if (tid == 0 && tab_flag[ta] != 0 && clip_status != nullptr) clip_status[t.k] = VP_EUNSUPPORTED;
    if (t.j != cur_j || t.s != cur_s) {
      // ---- K2 for this slice: union window of my column pair, f64 Keys / f64 sums -> fp32 ----
      cur_j = t.j;
      cur_s = t.s;
      const int q = warp * 32 + lane;
      hact = 2 * q < jn;
      const int ja = j0 + 2 * min(q, max(jn / 2 - 1, 0));
      const Win w0 = window_of(pl.in_w, pl.out_w, ja);
      const Win w1 = window_of(pl.in_w, pl.out_w, ja + 1);
      double s0 = 0.0, s1 = 0.0;
      for (int x = w0.x0; x < w0.x1; ++x) s0 += keys_d(((double)x - w0.c + 0.5) * w0.inv);
      for (int x = w1.x0; x < w1.x1; ++x) s1 += keys_d(((double)x - w1.c + 0.5) * w1.inv);
      const double r0 = s0 != 0.0 ? s0 : 1.0, r1 = s1 != 0.0 ? s1 : 1.0;
      const int xu = min(w0.x0, w1.x0);
      if (hact && max(w0.x1, w1.x1) - xu > kUL && clip_status != nullptr) clip_status[t.k] = VP_EUNSUPPORTED;
#pragma unroll
      for (int u = 0; u < kUL; ++u) {
        const int x = xu + u;
        const float wa = (x >= w0.x0 && x < w0.x1) ? (float)(keys_d(((double)x - w0.c + 0.5) * w0.inv) / r0) : 0.f;
        const float wb = (x >= w1.x0 && x < w1.x1) ? (float)(keys_d(((double)x - w1.c + 0.5) * w1.inv) / r1) : 0.f;
        wp[u] = make_float2(wa, wb);
        toff[u] = buf_s + (uint32_t)tpos(x - pa) * 16u;
      }
      const int jl0 = ja % B, wbk = ja / B, mw = jl0 / p, px = jl0 - mw * p;
      colpart = (wbk * m * m + mw) * D + px;
    }
    // ---- output addressing of frame f (O7, O8): element (row, q) of pixel_values at row*D + q ----
    void* pv = pl.is_image ? pv_img : pv_vid;
    const int64_t cap = pl.is_image ? img_cap : vid_cap;
    const bool writable = pv != nullptr && pl.patch_offset + (int64_t)pl.grid_t * pl.grid_h * pl.grid_w <= cap;
    const bool hst = writable && hact;
    const int f = t.f;
    const int last_slot = (f == pl.n_frames - 1) ? pl.grid_t * tp - 1 : f;     // frame n-1 fills the pad slots
    const int nslots = last_slot - f + 1;
    const int g0 = f / tp, ti0 = f - g0 * tp;
    const int64_t group_stride = (int64_t)(pl.grid_h / m) * (pl.grid_w / m) * m * m * D;
    const int hb_stride = (pl.grid_w / m) * m * m * D;        // one merge-row band of one temporal group
    // this lane's first element of frame f's slot: row offsets are added per output row
    char* const lbase = reinterpret_cast<char*>(pv) +
        (pl.patch_offset * (int64_t)D + (int64_t)g0 * group_stride + (int64_t)ti0 * p * p + colpart) * kEsz;

    float4 acc[4][3];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int q = 0; q < 3; ++q) acc[r][q] = make_float4(0.f, 0.f, 0.f, 0.f);
    // byte offset of this lane's 12 bytes inside a staged row (the part starts at (3*pa) & 15)
    const uint32_t lofs = (uint32_t)(((3 * pa) & 15) + 12 * lane);

    int y = 0;
    // one source row into the ring (output row ib+U being completed sits in slot U)
    // staged row rc: bytes n0..n2 and weight record wv (after its group's TMA landed)
    uint32_t n0, n1, n2;
    float4 wv;
    auto load_row = [&]() {
      if ((rc & (kTGrp - 1)) == 0) mbar_wait(&full[(rc / kTGrp) % kTNGrp], (rc / kTDepth) & 1);
      const uint32_t slot = rc % kTDepth;
      const uint32_t sa = stage_s + slot * kTRowB + lofs;
      n0 = lds_u32(sa); n1 = lds_u32(sa + 4); n2 = lds_u32(sa + 8);
      wv = lds_f4(wrec_s + slot * 16);
    };
    if (VP_TEAM_PF) load_row();
#define VP_TEAM_BODY(U)                                                                                      \
    {                                                                                                         \
      if (!VP_TEAM_PF) load_row();                                                                            \
      const uint32_t slot = rc % kTDepth;                                                                     \
      float2 fv[6];                                                                                           \
      cvt_i2f(n0, fv[0], fv[1]);                                                                              \
      cvt_i2f(n1, fv[2], fv[3]);                                                                              \
      cvt_magic(n2, fv[4], fv[5]);                                                                            \
      const float4 wc = wv;                                                                                   \
      ++rc;                                                                                                   \
      if ((slot & (kTGrp - 1)) == kTGrp - 1) {                                                                \
        __syncwarp();                                                                                         \
        issue_group(slot / kTGrp);                                                                            \
      }                                                                                                       \
      if (VP_TEAM_PF) load_row();                                                                             \
      ring4<U>(acc, wc, fv);                                                                                  \
    }

    // retire output row i = ib + U from slot U into buffer U & 1, barrier, H of row i.  Row offset of output
    // row i (O8): (i / (m p)) * hb_stride + ((i / p) % m) * m * D + (i % p) * p; for the preset (p % 4 == 0) the
    // 4 rows of a group share i / p, so row ib+U is the group's offset + U*p (an immediate).
#define VP_TEAM_RETIRE(U)                                                                                    \
    {                                                                                                         \
      const uint32_t ra = vsa + (U & 1) * kTPx * 16;                                                          \
      const float4* a = acc[U];                                                                               \
      sts_f4(ra, a[0]);                                                                                       \
      sts_f4(ra + 128, make_float4(a[0].w, a[1].x, a[1].y, 0.f));                                             \
      sts_f4(ra + 256, make_float4(a[1].z, a[1].w, a[2].x, a[2].y));                                          \
      sts_f4(ra + 384, make_float4(a[2].y, a[2].z, a[2].w, 0.f));                                             \
      _Pragma("unroll") for (int q = 0; q < 3; ++q) acc[U][q] = make_float4(0.f, 0.f, 0.f, 0.f);              \
      __syncthreads();                                                                                        \
      if (hst) {                                                                                              \
        float2 ar = make_float2(0.f, 0.f), ag = ar, ab = ar;                                                  \
        _Pragma("unroll") for (int u = 0; u < kUL; ++u) {                                                     \
          const float4 v = lds_f4(toff[u] + (U & 1) * kTPx * 16);                                             \
          ar = __ffma2_rn(make_float2(v.x, v.x), wp[u], ar);                                                  \
          ag = __ffma2_rn(make_float2(v.y, v.y), wp[u], ag);                                                  \
          ab = __ffma2_rn(make_float2(v.z, v.z), wp[u], ab);                                                  \
        }                                                                                                     \
        const int i = ib + U;                                                                                 \
        const int ro = (P > 0 && (P & 3) == 0) ? ro_grp + U * p                                               \
                                               : (i / B) * hb_stride + ((i / p) % m) * m * D + (i % p) * p;  \
        store_pair<kF32>(kp, lbase + (int64_t)ro * kEsz, ar, ag, ab, cstride, nslots, ti0, tp, p, group_stride);\
      }                                                                                                       \
    }

    int4 ye_next = __ldg(reinterpret_cast<const int4*>(y1));
    for (int ib = 0; ib < out_h; ib += 4) {
      const int4 ye = ye_next;                    // window ends of rows ib..ib+3, prefetched one group ahead
      if (ib + 4 < out_h) ye_next = __ldg(reinterpret_cast<const int4*>(y1 + ib + 4));
      const int ro_grp = (ib / B) * hb_stride + ((ib / p) % m) * m * D + (ib % p) * p;
#define VP_TEAM_ROW(U, YE)                                                                                   \
      if (ib + U < out_h) {                                                                                   \
        const int yend = YE;                                                                                  \
        for (; y < yend; ++y) VP_TEAM_BODY(U)                                                                 \
        VP_TEAM_RETIRE(U)                                                                                     \
      }
      VP_TEAM_ROW(0, ye.x)
      VP_TEAM_ROW(1, ye.y)
      VP_TEAM_ROW(2, ye.z)
      VP_TEAM_ROW(3, ye.w)
#undef VP_TEAM_ROW
    }
    // source rows below the last window (zero weights): keep the staging ring in step
    for (; y < in_h; ++y) {
      if (!VP_TEAM_PF && (rc & (kTGrp - 1)) == 0) mbar_wait(&full[(rc / kTGrp) % kTNGrp], (rc / kTDepth) & 1);
      const uint32_t slot = rc % kTDepth;
      ++rc;
      if ((slot & (kTGrp - 1)) == kTGrp - 1) {
        __syncwarp();
        issue_group(slot / kTGrp);
      }
      if (VP_TEAM_PF && (rc & (kTGrp - 1)) == 0) mbar_wait(&full[(rc / kTGrp) % kTNGrp], (rc / kTDepth) & 1);
    }
#undef VP_TEAM_BODY
#undef VP_TEAM_RETIRE
  }
}


// ---------------------------------------------------------------- per-clip vertical tables (K2 for KV_TEAM)
// y1tab[j][i] = end of output row i's window (padded with in_h to a multiple of 4); vtab[j][y] = fp32 weights
// (f64 Keys / f64 window sum, C10) of the output rows i(y)..i(y)+3, i(y) = first output row with y1 > y: the row
// the kernel is completing when it consumes source row y.  One table per run of equal (in_h, out_h) in the list.
__device__ __forceinline__ double win_sum(const Win& w) {
  double s = 0.0;
  for (int x = w.x0; x < w.x1; ++x) s += keys_d(((double)x - w.c + 0.5) * w.inv);
  return s;
}

__global__ void __launch_bounds__(128)
team_vtab_kernel(const vp_clip_plan* __restrict__ plans, const VIdx vx, const int* __restrict__ alias,
                 float4* __restrict__ vtab, int* __restrict__ y1tab, int* __restrict__ tflag) {
  const int j = blockIdx.y;
  if (j >= (int)vx.meta[0] || alias[j] != j) return;
  const vp_clip_plan& pl = plans[vx.list[j]];
  const int in_h = pl.in_h, out_h = pl.out_h;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < ((out_h + 3) & ~3)) y1tab[(int64_t)j * kTabOutH + r] = r < out_h ? window_of(in_h, out_h, r).x1 : in_h;
  if (r >= in_h) return;
  const int y = r;
  const double s = (double)in_h / (double)out_h;
  const double sup = 2.0 * (s > 1.0 ? s : 1.0);
  int i = (int)floor(((double)y - sup - 0.5) / s - 0.5);
  i = max(0, min(i, out_h));
  while (i > 0 && window_of(in_h, out_h, i - 1).x1 > y) --i;
  while (i < out_h && window_of(in_h, out_h, i).x1 <= y) ++i;
  float wv[4] = {0.f, 0.f, 0.f, 0.f};
  for (int q = 0; q < 5 && i + q < out_h; ++q) {
    const Win w = window_of(in_h, out_h, i + q);
    if (w.x0 > y) break;
    const double sum = win_sum(w);
    const double wt = keys_d(((double)y - w.c + 0.5) * w.inv) / (sum != 0.0 ? sum : 1.0);
    if (q < 4) wv[q] = (float)wt;
    else if (fabs(wt) > 1e-9) atomicOr(&tflag[j], 1);     // a 5th live row with a non-negligible weight
  }
  vtab[(int64_t)j * kTabInH + y] = make_float4(wv[0], wv[1], wv[2], wv[3]);
}

// ---------------------------------------------------------------- per-variant work index
// One CTA: slot v in {MILD, MEDIUM, STRONG, COPY, TEAM} collects the valid, 16-B aligned clips of that variant
// (list, batch order) and the exclusive prefix of their item counts (off); meta[v] = {count, items}.  For the
// TEAM list, alias[j] = first position of the run of equal (in_h, out_h) that j belongs to (shared tables).
constexpr int kIdxThreads = 1024;
__device__ __forceinline__ int variant_slot(int kv) {
  return kv == KV_COPY ? 3 : (kv == KV_TEAM ? 4 : (kv <= KV_STRONG ? kv : -1));
}

__global__ void __launch_bounds__(kIdxThreads)
variant_index_kernel(const vp_clip_plan* __restrict__ plans, int n, const int64_t* __restrict__ coff,
                     const int64_t* __restrict__ pitch, int* __restrict__ list, int64_t* __restrict__ off,
                     int64_t* __restrict__ meta, int* __restrict__ alias, int* __restrict__ tflag) {
  __shared__ int64_t wsum[kIdxThreads / 32][kNSlots];
  __shared__ int wcnt[kIdxThreads / 32][kNSlots];
  __shared__ int64_t c_items[kNSlots];
  __shared__ int c_cnt[kNSlots];
  __shared__ int wmax[kIdxThreads / 32];
  __shared__ int c_alias;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < kNSlots) { c_items[tid] = 0; c_cnt[tid] = 0; }
  if (tid == 0) c_alias = 0;
  __syncthreads();
  for (int c0 = 0; c0 < n; c0 += kIdxThreads) {
    const int k = c0 + tid;
    int slot = -1;
    int64_t items = 0;
    if (k < n) {
      const vp_clip_plan& pl = plans[k];
      if (pl.status == VP_OK && pl.tile_count > 0 && ((coff[k] | pitch[k]) & 15) == 0) {
        slot = variant_slot(pl.kernel_variant);
        items = pl.tile_count;
      }
    }
    int64_t ex_items = 0;
    int ex_cnt = 0;
#pragma unroll
    for (int v = 0; v < kNSlots; ++v) {
      int64_t x = slot == v ? items : 0;
      int y = slot == v ? 1 : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t xa = __shfl_up_sync(0xffffffffu, x, o);
        const int ya = __shfl_up_sync(0xffffffffu, y, o);
        if (lane >= o) { x += xa; y += ya; }
      }
      if (lane == 31) { wsum[warp][v] = x; wcnt[warp][v] = y; }
      if (slot == v) { ex_items = x - items; ex_cnt = y - 1; }
    }
    __syncthreads();
    int64_t add_items = 0, tot_items[kNSlots];
    int add_cnt = 0, tot_cnt[kNSlots];
#pragma unroll
    for (int v = 0; v < kNSlots; ++v) { tot_items[v] = 0; tot_cnt[v] = 0; }
    for (int w = 0; w < kIdxThreads / 32; ++w) {
#pragma unroll
      for (int v = 0; v < kNSlots; ++v) {
        if (w < warp && slot == v) { add_items += wsum[w][v]; add_cnt += wcnt[w][v]; }
        tot_items[v] += wsum[w][v];
        tot_cnt[v] += wcnt[w][v];
      }
    }
    if (slot >= 0) {
      const int pos = c_cnt[slot] + add_cnt + ex_cnt;
      list[(size_t)slot * n + pos] = k;
      off[(size_t)slot * (n + 1) + pos] = c_items[slot] + add_items + ex_items;
    }
    __syncthreads();
    if (tid < kNSlots) { c_items[tid] += tot_items[tid]; c_cnt[tid] += tot_cnt[tid]; }
    __syncthreads();
  }
  if (tid < kNSlots) {
    off[(size_t)tid * (n + 1) + c_cnt[tid]] = c_items[tid];
    meta[2 * tid] = c_cnt[tid];
    meta[2 * tid + 1] = c_items[tid];
  }
  __syncthreads();
  // TEAM table aliases: inclusive max-scan of run starts over the TEAM list
  const int nt = c_cnt[4];
  const int* tl = list + (size_t)4 * n;
  for (int c0 = 0; c0 < nt; c0 += kIdxThreads) {
    const int j = c0 + tid;
    int v = -1;
    if (j < nt) {
      tflag[j] = 0;
      const vp_clip_plan& a = plans[tl[j]];
      bool start = j == 0;
      if (!start) {
        const vp_clip_plan& b = plans[tl[j - 1]];
        start = a.in_h != b.in_h || a.out_h != b.out_h;
      }
      v = start ? j : -1;
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) v = max(v, __shfl_up_sync(0xffffffffu, v, o));
    if (lane == 31) wmax[warp] = v;
    __syncthreads();
    int pre = c_alias;
    for (int w = 0; w < warp; ++w) pre = max(pre, wmax[w]);
    if (j < nt) alias[j] = max(pre, v);
    __syncthreads();
    if (tid == kIdxThreads - 1) c_alias = max(pre, v);
    __syncthreads();
  }
}

// Per-device one-time setup (thread-safe: attribute calls are idempotent, the bits only skip repeats).
constexpr int kMaxDev = 64;
std::atomic<int> g_sms[kMaxDev];

}  // namespace

int device_sms(int dev) {
  if (dev < 0 || dev >= kMaxDev) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
  }
  int n = g_sms[dev].load(std::memory_order_relaxed);
  if (n <= 0) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    g_sms[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

// Caller workspace of vp_resize_normalize_patchify: the work index and the KV_TEAM tables.
ResizeWs resize_ws_layout(int n, void* base) {
  ResizeWs w{};
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o = (o + bytes + 255) & ~(size_t)255;
    return at;
  };
  const size_t o_list = take((size_t)kNSlots * n * sizeof(int));
  const size_t o_off = take((size_t)kNSlots * (n + 1) * sizeof(int64_t));
  const size_t o_meta = take(2 * kNSlots * sizeof(int64_t));
  const size_t o_alias = take((size_t)n * sizeof(int));
  const size_t o_flag = take((size_t)n * sizeof(int));
  const size_t o_vtab = take((size_t)n * kTabInH * sizeof(float4));
  const size_t o_y1 = take((size_t)n * kTabOutH * sizeof(int));
  w.bytes = o;
  char* b = reinterpret_cast<char*>(base);
  if (b != nullptr) {
    w.list = reinterpret_cast<int*>(b + o_list);
    w.off = reinterpret_cast<int64_t*>(b + o_off);
    w.meta = reinterpret_cast<int64_t*>(b + o_meta);
    w.alias = reinterpret_cast<int*>(b + o_alias);
    w.tflag = reinterpret_cast<int*>(b + o_flag);
    w.vtab = reinterpret_cast<float4*>(b + o_vtab);
    w.y1tab = reinterpret_cast<int*>(b + o_y1);
  }
  return w;
}

VIdx ws_vidx(const ResizeWs& w, int n, int slot) {
  return VIdx{w.list + (size_t)slot * n, w.off + (size_t)slot * (n + 1), w.meta + 2 * slot};
}

cudaError_t launch_index(const vp_clip_plan* plans, int n, const int64_t* coff, const int64_t* pitch,
                         const ResizeWs& w, cudaStream_t s) {
  variant_index_kernel<<<1, kIdxThreads, 0, s>>>(plans, n, coff, pitch, w.list, w.off, w.meta, w.alias, w.tflag);
  return cudaGetLastError();
}

cudaError_t launch_team(const FKParams& kp, const vp_clip_plan* plans, int n, const ResizeWs& w, const uint8_t* frames,
                        const int64_t* coff, const int64_t* pitch, void* pi, int64_t icap, void* pvv, int64_t vcap,
                        int32_t* clip_status, int num_sms, cudaStream_t s) {
  const VIdx vx = ws_vidx(w, n, 4);
  dim3 tg((kTabInH + 127) / 128, n);
  team_vtab_kernel<<<tg, 128, 0, s>>>(plans, vx, w.alias, w.vtab, w.y1tab, w.tflag);
  const bool preset = kp.p == 16 && kp.m == 2 && kp.tp == 2;       // Qwen2.5/3-VL geometry: compile-time addressing
  auto kern = kp.out_f32 ? (preset ? resize_team_kernel<kTeamUL, true, 16, 2, 2> : resize_team_kernel<kTeamUL, true, 0, 0, 0>)
                         : (preset ? resize_team_kernel<kTeamUL, false, 16, 2, 2> : resize_team_kernel<kTeamUL, false, 0, 0, 0>);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kTT, 0);
  if (per_sm < 1) per_sm = 1;
  kern<<<num_sms * per_sm, kTT, 0, s>>>(kp, plans, vx, w.alias, w.tflag, w.vtab, w.y1tab, frames, coff, pitch, pi, icap,
                                        pvv, vcap, clip_status);
  return cudaGetLastError();
}

}  // namespace vp
