// vp_resize_team.cu -- K3 team kernels (KV_TEAM, KV_WIDE): streaming fused AA-bicubic resize + clamp + normalise +
// temporal pad + patchify (O4-O9) for downscales / identity on both axes with a narrow horizontal window.
//
// Work item = (clip, slice, source frame f).  A slice is a range of output columns whose source footprint fits the
// CTA's NV*128 pixels (KV_WIDE: the whole frame row).  A CTA of NV V warps + NH H warps walks the item's source rows
// top to bottom exactly once:
//   V warps: warp v owns a 128-pixel (384-byte) part of the footprint; lane L converts its 12 bytes (4 RGB pixels) of
//      each staged source row once (I2F.U8 on the XU pipe for 2 of 3 words, PRMT + FADD2 for the third: both exact)
//      and FMAs them (FFMA2, broadcast weight) into a 4-slot register ring of live output rows.  For a downscale
//      (in >= out) at most 4 output rows are live at any source row (window 4s wide, centres s apart),
//      so 4 slots carry no dead FMAs at the bench ratio.  Output row i lives in ring slot i % 4 and each source
//      row's weight record is stored in slot order, so the FMAs of every row use static slots; the rows of a staging
//      group are walked in pairs with the next row's loads issued ahead.  A finished row (switch on i % 4) is stored
//      (float4 RGB + pad per pixel, conflict-free layout rpos) into one of kNR retire slots: wait until the H warps
//      released the slot (mbarrier rempty), store, arrive on rfull.
//   H warps: lane (warp h, lane l) owns output column pairs q = 32h + l (+ 32 NH per further pair) of the slice; the
//      pair's union window (<= kUL taps; weights (w_a, w_b) and the taps' shared addresses in registers for the whole
//      slice) is read once per row (LDS.128) and FMA'd as 3 FFMA2 (pixel channel broadcast x pair weights);
//      normalise, clamp in the output domain, pack bf16x2 / float2 and store straight into the HF patch layout, once
//      per temporal slot the frame fills (O7); then release the retire slot.
//
// Staging: the CTA's source rows land in a kTDepth-row shared ring by cp.async.bulk, refilled in groups of kTGrp rows
// (one mbarrier per group) by the last V warp to finish a group; when the copied span of a row is the whole row
// pitch (KV_WIDE frames packed at their pitch, e.g. cfg5) a group that does not start an item is one contiguous bulk
// copy, its rows at stride pitch.  The vertical weights travel with the rows: per
// source row a 16-B record (the fp32 weights of its <= 4 live output rows, in ring-slot order) copied by TMA from the
// per-clip table that team_vtab_kernel writes into the caller's workspace (f64 Keys / f64 window sum -> fp32, C10).
// Consecutive clips of equal (in_h, out_h) share one table.
#include "vp_k3_common.cuh"
#include <atomic>
#include <type_traits>

namespace vp {
namespace {

#ifndef VP_TEAM_DEPTH
#define VP_TEAM_DEPTH 16
#endif
constexpr int kTDepth = VP_TEAM_DEPTH;      // staged source rows per V warp
#ifndef VP_TEAM_GRP
#define VP_TEAM_GRP 8
#endif
constexpr int kTGrp = VP_TEAM_GRP;          // rows per refill group (one mbarrier phase)
constexpr int kTNGrp = kTDepth / kTGrp;
#ifndef VP_TEAM_NR
#define VP_TEAM_NR 4
#endif
constexpr int kNR = VP_TEAM_NR;             // retire slots (rows V may run ahead of H); a multiple of 4
#ifndef VP_TEAM_HINT
#define VP_TEAM_HINT 0      // suspend-time hint (ns) of the V<->H retire-slot waits; 0 = spin
#endif
// Verification build only (scripts/sanitize.sh): every lane arrives on the retire-slot barriers instead of lane 0
// after __syncwarp (equivalent under the PTX memory model -- bar.warp.sync orders the warp's shared-memory writes
// before lane 0's release -- but compute-sanitizer racecheck only credits a thread's own arrive).
#ifndef VP_ALL_LANES_ARRIVE
#define VP_ALL_LANES_ARRIVE 0
#endif

template <int NV, int NH, bool kLarge = false>
struct SplitCfg {
  static constexpr int kPx = NV * 128;                                    // footprint pixels per CTA
  // retire-slot stride in pixels: KV_TEAML keeps rows unswizzled with kTeamULL zero pixels of tail padding, so every
  // tap of a pair window is base + 16 u (no per-tap address registers, no clamping)
  static constexpr int kPxPad = kLarge ? kPx + kTeamULL : kPx;
  static constexpr int kThreads = (NV + NH) * 32;
  // staged row: footprint + alignment slack (KV_WIDE's single slice starts at pixel 0: no slack)
  static constexpr int kRowB = NV == kWideNV ? NV * 384 : (NV * 384 + 16 + 15) & ~15;
  static constexpr size_t OFF_STG = 0;
  static constexpr size_t OFF_WREC = OFF_STG + (size_t)kTDepth * kRowB;
  static constexpr size_t OFF_BUF = OFF_WREC + (size_t)kTDepth * 16;
  static constexpr size_t OFF_SBAR = OFF_BUF + (size_t)kNR * kPxPad * 16;
  static constexpr size_t OFF_RBAR = OFF_SBAR + (size_t)kTNGrp * 8;
  static constexpr size_t OFF_CNT = OFF_RBAR + (size_t)2 * kNR * 8;
  static constexpr size_t OFF_PROD = (OFF_CNT + (size_t)kTNGrp * 4 + 15) & ~(size_t)15;
  static constexpr size_t OFF_EBAR = OFF_PROD + 48;   // staging "read" barriers (VP_ALL_LANES_ARRIVE build only)
  static constexpr size_t SMEM = OFF_EBAR + (size_t)kTNGrp * 8;
  static_assert(OFF_WREC % 16 == 0 && OFF_BUF % 16 == 0 && OFF_SBAR % 8 == 0 && OFF_PROD % 16 == 0, "align");
};

// Producer state of the CTA's staging ring (shared memory; read and updated only by the V warp that refills a
// group -- refills are serialised because the last reader of group g+1 starts after the refill of g was issued).
struct TeamProd {
  const uint8_t* src;       // next source row of the CTA footprint (16-B aligned down)
  const float4* wr;         // its weight record
  int64_t pitch;
  int64_t next;             // next item to open
  int rows, nbytes;         // rows left in the current item, bytes copied per row
};
static_assert(sizeof(TeamProd) <= 48, "TeamProd");

struct TItem {
  int j;                    // position in the variant list
  int k;                    // clip index
  int s, f;                 // slice, frame
  int ws;                   // slice width
  int r0, r1;               // output rows of the item's band [r0, r1) (the whole frame unless the launch is banded)
};

template <int NV, int NH, bool kBand>
__device__ __forceinline__ TItem decode_item(const VIdx& vx, int cnt, int64_t item, const vp_clip_plan* plans, int p) {
  TItem t;
  t.j = vfind(vx, cnt, item);
  t.k = vx.list[t.j];
  const vp_clip_plan& pl = plans[t.k];
  t.ws = team_geometry(pl.in_w, pl.out_w, p, NV, NH).ws;
  const int64_t local = item - vx.off[t.j];
  if (!kBand) {
    t.s = (int)(local / pl.n_frames);          // slice-major: consecutive items share the slice's H weights
    t.f = (int)(local - (int64_t)t.s * pl.n_frames);
    t.r0 = 0;
    t.r1 = pl.out_h;
    return t;
  }
  const int nb = (int)vx.meta[2];
  const int nbd = band_count(pl.out_h, nb), bs = band_rows(pl.out_h, nb);
  const int64_t per_slice = (int64_t)pl.n_frames * nbd;
  t.s = (int)(local / per_slice);
  const int rem = (int)(local - (int64_t)t.s * per_slice);
  const int b = rem / pl.n_frames;
  t.f = rem - b * pl.n_frames;
  t.r0 = b * bs;
  t.r1 = min(pl.out_h, t.r0 + bs);
  return t;
}

// Source rows [ys, ye) of a band: from the first row of output row r0's window to the end of row r1-1's window.
__device__ __forceinline__ int band_ys(const vp_clip_plan& pl, int r0) {
  return r0 == 0 ? 0 : window_of(pl.in_h, pl.out_h, r0).x0;
}

// Slice span: output columns [j0, j0+jn), footprint pixels [pa, pa+np) with pa a multiple of 4.
__device__ __forceinline__ void slice_span(const vp_clip_plan& pl, int ws, int s, int& j0, int& jn, int& pa, int& np) {
  j0 = s * ws;
  jn = min(ws, pl.out_w - j0);
  pa = window_of(pl.in_w, pl.out_w, j0).x0 & ~3;
  np = window_of(pl.in_w, pl.out_w, j0 + jn - 1).x1 - pa;
}

__device__ __forceinline__ float2& h2(float4& v, int h) { return reinterpret_cast<float2*>(&v)[h]; }

// Retired-row layout (KV_WIDE / KV_TEAM): pixel-major float4, granule class (x + 5 (x >> 3)) mod 8 inside each
// 8-pixel block.  V retire stores (lane L writes pixels 4L..4L+3, one per instruction) are conflict-free (4 per-lane
// offsets), and each H lane walks its union window in a rotated order -- at tap tt every lane reads a row position
// = tt (mod UL); weights and addresses are rotated at slice setup -- so the H tap reads are conflict-free too: 1.00
// wavefront per quarter-warp at every ratio simulated, vs 1.35 for round 1's sub-pixel-major swizzle at the cfg2
// ratio (scripts/bank_sim.py); cfg5 K3 6.89 -> 6.34 ms per 64 clips.
__device__ __forceinline__ int rpos(int x) { return (x & ~7) | ((x + 5 * (x >> 3)) & 7); }


// A lane's 12 staged bytes (R0 G0 B0 R1 | G1 B1 R2 G2 | B2 R3 G3 B3 in words n0, n1, n2) as the six FFMA2 operand
// pairs of the ring, ordered so that the accumulator quads are (R0 G0 B0 R3), (R1 G1 B1 G3), (R2 G2 B2 B3): pixels
// 0..2 retire as whole quads (their .w is pixel 3's channel, ignored by the horizontal pass) and pixel 3 is the .w
// column.  8 bytes convert on the XU pipe (I2F.U8 with a byte select), 4 on ALU + FMA (PRMT + FADD2).
__device__ __forceinline__ float byte_i2f(uint32_t w, int k) { return (float)((w >> (8 * k)) & 0xffu); }
__device__ __forceinline__ float byte_magic(uint32_t w, int k) {      // 2^23 + b (exact)
  return __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7540u + (unsigned)k));
}
__device__ __forceinline__ void cvt_ring(uint32_t n0, uint32_t n1, uint32_t n2, float2 (&f)[6]) {
  const float2 mm = make_float2(-8388608.f, -8388608.f);
  f[0] = make_float2(byte_i2f(n0, 0), byte_i2f(n0, 1));                                   // R0 G0
  f[1] = __fadd2_rn(make_float2(byte_magic(n0, 2), byte_magic(n2, 1)), mm);               // B0 R3
  f[2] = make_float2(byte_i2f(n0, 3), byte_i2f(n1, 0));                                   // R1 G1
  f[3] = __fadd2_rn(make_float2(byte_magic(n1, 1), byte_magic(n2, 2)), mm);               // B1 G3
  f[4] = make_float2(byte_i2f(n1, 2), byte_i2f(n1, 3));                                   // R2 G2
  f[5] = make_float2(byte_i2f(n2, 0), byte_i2f(n2, 3));                                   // B2 B3
}

// normalise (O6) as FFMA2 over the column pair, clamp (C12) in the output domain (clamp(v,0,255)*s+b ==
// clamp(v*s+b, lo, hi) with lo/hi the images of 0 and 255, ordered), round (O9) and store the pair into every
// temporal slot the frame fills (O7); for bf16 RNE is monotone, so clamping the rounded pair is bit-identical.
template <bool kF32, bool kFold>
__device__ __forceinline__ void store_pair(const FKParams& kp, char* q, float2 ar, float2 ag, float2 ab, int cstride,
                                           int nslots, int ti0, int tp, int p, int64_t group_stride) {
  constexpr int kEsz = kF32 ? 4 : 2;
  // kFold: the pair weights carry the (channel-uniform) scale and the accumulators start at the bias, so the sums
  // are already normalised
  const float2 n[3] = {kFold ? ar : __ffma2_rn(ar, make_float2(kp.scale[0], kp.scale[0]), make_float2(kp.bias[0], kp.bias[0])),
                       kFold ? ag : __ffma2_rn(ag, make_float2(kp.scale[1], kp.scale[1]), make_float2(kp.bias[1], kp.bias[1])),
                       kFold ? ab : __ffma2_rn(ab, make_float2(kp.scale[2], kp.scale[2]), make_float2(kp.bias[2], kp.bias[2]))};
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

template <int NV, int NH, int PPL, int kUL, bool kF32, bool kFold, int P, int M, int TP, int MINB, bool kLarge, bool kBand>
__global__ void __launch_bounds__((NV + NH) * 32, MINB)
resize_split_kernel(FKParams kp, const vp_clip_plan* __restrict__ plans, const VIdx vx, const int* __restrict__ tab_alias,
                    const int* __restrict__ tab_flag, const float4* __restrict__ vtab, const int* __restrict__ y1tab,
                    const uint8_t* __restrict__ frames, const int64_t* __restrict__ clip_off,
                    const int64_t* __restrict__ pitch_arr, void* pv_img, int64_t img_cap, void* pv_vid, int64_t vid_cap,
                    int32_t* __restrict__ clip_status) {
  using Cfg = SplitCfg<NV, NH, kLarge>;
  constexpr int kPx = Cfg::kPx;
  static_assert(!kLarge || (PPL == 1 && kUL <= kTeamULL), "KV_TEAML: one pair per lane, padded rows");
  auto pos = [](int x) { return kLarge ? x : (rpos(x)); };   // retired-row pixel position
  constexpr int kRowB = Cfg::kRowB;
  // preset geometry (p % 4 == 0 and p*m % 4 == 0): every out_h is a multiple of 4, so with 4 retire slots the slot of
  // output row i is i % 4 = the static unroll index U
  constexpr bool kStatic = P > 0 && (P % 4) == 0 && ((P * M) % 4) == 0 && (kNR % 4) == 0;
  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  int lane;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(lane));
  const bool l0 = lane == 0;
  const int p = P > 0 ? P : kp.p, m = P > 0 ? M : kp.m, tp = P > 0 ? TP : kp.tp;

  // kBand: the instantiation for launches cut into row bands (variant_index_kernel's meta[2] > 1); both are launched
  // and the one that does not match exits here, so the whole-frame path carries no band bookkeeping
  if ((vx.meta[2] > 1) != kBand) return;
  const int cnt = (int)vx.meta[0];
  const int64_t total = vx.meta[1];
  const int64_t my_a = total * blockIdx.x / gridDim.x;
  const int64_t my_b = total * (blockIdx.x + 1) / gridDim.x;
  if (my_a >= my_b) return;

  uint8_t* stage = smem + Cfg::OFF_STG;
  float4* wrec = reinterpret_cast<float4*>(smem + Cfg::OFF_WREC);
  uint64_t* sfull = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_SBAR);      // staging group landed (TMA tx)
  uint64_t* rfull = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_RBAR);      // V -> H: retire slot filled
  uint64_t* rempty = rfull + kNR;                                           // H -> V: retire slot released
  int* gcnt = reinterpret_cast<int*>(smem + Cfg::OFF_CNT);                  // V warps done with a staging group
  uint64_t* sread = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_EBAR);      // verification build: group read
  TeamProd* ps = reinterpret_cast<TeamProd*>(smem + Cfg::OFF_PROD);
  float4* buf0 = reinterpret_cast<float4*>(smem + Cfg::OFF_BUF);
  const uint32_t buf_s = smem_u32(buf0);
  constexpr uint32_t kSlotB = (uint32_t)Cfg::kPxPad * 16;   // bytes per retire slot

  // ---- staging producer: refill group g with the next kTGrp source rows of the CTA's item sequence (warp-uniform
  //      caller; the copies and barrier operations are predicated to lane 0) ----
  auto open_item = [&](TeamProd& st) {
    const TItem t = decode_item<NV, NH * PPL, kBand>(vx, cnt, st.next, plans, p);
    const vp_clip_plan& pl = plans[t.k];
    int j0, jn, pa, np;
    slice_span(pl, t.ws, t.s, j0, jn, pa, np);
    const int b0 = 3 * pa, o = b0 & 15;
    const int ys = kBand ? band_ys(pl, t.r0) : 0;
    const int ye = kBand ? __ldg(y1tab + (int64_t)tab_alias[t.k] * kTabOutStride + t.r1 - 1) : pl.in_h;
    st.nbytes = (o + 3 * np + 15) & ~15;
    st.pitch = pitch_arr[t.k];
    st.src = frames + clip_off[t.k] + ((int64_t)t.f * pl.in_h + ys) * st.pitch + (b0 - o);
    st.wr = vtab + (int64_t)tab_alias[t.k] * kTabInH + ys;
    st.rows = ye - ys;
    ++st.next;
  };
  auto issue_group = [&](uint32_t g) {
    asm volatile("mov.b32 %0, %0;" : "+r"(g));   // opaque copy (nvcc 12.9 mbarrier-address CSE workaround)
    TeamProd st = *ps;
    if (st.rows >= kTGrp) {
      mbar_expect_tx_if(&sfull[g], (uint32_t)(kTGrp * st.nbytes + kTGrp * 16), l0);
      if (st.pitch == st.nbytes) {
        // the copied span of each row is the whole row pitch: the group's rows are one contiguous block, one bulk copy
        // (rows land at stride pitch <= kRowB; the V warps address whole groups at that stride)
        tma_bulk_g2s_if(stage + (size_t)(g * kTGrp) * kRowB, st.src, (uint32_t)(kTGrp * st.nbytes), &sfull[g], l0);
      } else {
#pragma unroll
        for (int q = 0; q < kTGrp; ++q)
          tma_bulk_g2s_if(stage + (size_t)(g * kTGrp + q) * kRowB, st.src + (int64_t)q * st.pitch, (uint32_t)st.nbytes,
                          &sfull[g], l0);
      }
      tma_bulk_g2s_if(wrec + g * kTGrp, st.wr, kTGrp * 16, &sfull[g], l0);
      st.src += (int64_t)kTGrp * st.pitch;
      st.wr += kTGrp;
      st.rows -= kTGrp;
    } else {
#pragma unroll 1
      for (int q = 0; q < kTGrp; ++q) {
        if (st.rows == 0 && st.next < my_b) open_item(st);
        if (st.rows > 0) {
          mbar_expect_tx_if(&sfull[g], (uint32_t)(st.nbytes + 16), l0);
          tma_bulk_g2s_if(stage + (size_t)(g * kTGrp + q) * kRowB, st.src, (uint32_t)st.nbytes, &sfull[g], l0);
          tma_bulk_g2s_if(wrec + g * kTGrp + q, st.wr, 16, &sfull[g], l0);
          st.src += st.pitch;
          st.wr += 1;
          --st.rows;
        }
      }
    }
    mbar_arrive_if(&sfull[g], l0);
    __syncwarp();
    if (l0) *ps = st;
    __syncwarp();
  };

  if (tid == 0) {
    for (int i = 0; i < kTNGrp; ++i) { mbar_init(&sfull[i], 1); mbar_init(&sread[i], NV * 32); gcnt[i] = 0; }
    for (int i = 0; i < kNR; ++i) {
      mbar_init(&rfull[i], VP_ALL_LANES_ARRIVE ? NV * 32 : NV);
      mbar_init(&rempty[i], VP_ALL_LANES_ARRIVE ? NH * 32 : NH);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    TeamProd z;
    z.src = nullptr; z.wr = nullptr; z.pitch = 0; z.next = my_a; z.rows = 0; z.nbytes = 0;
    *ps = z;
  }
  for (int i = tid; i < kNR * Cfg::kPxPad; i += Cfg::kThreads) buf0[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  __syncthreads();
  if (warp == 0)
    for (uint32_t g = 0; g < kTNGrp; ++g) issue_group(g);   // prefill

  if (warp < NV) {
    // ================================================================= V warps
    // The source-row loop runs over whole staging groups (kTGrp rows, fully unrolled: static staging offsets, the
    // group wait / refill once per group, and the next row's loads free to move above this row's FMAs).  Ring slot
    // s holds the output rows i with i % 4 == s and the weight records are stored in slot order (team_vtab_kernel),
    // so every row's FMAs use static slots; a row that completes output row i retires slot i % 4 (a switch, taken
    // once per output row).
    const uint32_t stage_s = smem_u32(stage), wrec_s = smem_u32(wrec);
    constexpr uint32_t kPxB = kLarge ? 16u : 128u;  // distance of the lane's consecutive pixels in the retired row
    constexpr bool kRot = !kLarge;
    uint32_t vo[4];                                  // retire addresses of the lane's 4 pixels in retire slot 0
    {
      const uint32_t vsa = buf_s + (uint32_t)pos(warp * 128 + lane * 4) * 16u;
#pragma unroll
      for (int j = 0; j < 4; ++j) vo[j] = kRot ? buf_s + (uint32_t)rpos(warp * 128 + lane * 4 + j) * 16u : vsa + j * kPxB;
    }
    float4 acc[4][3];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int q = 0; q < 3; ++q) acc[r][q] = make_float4(0.f, 0.f, 0.f, 0.f);
    uint32_t rc = 0;                              // staged rows consumed (a multiple of kTGrp at every group start)
    uint32_t rr = 0;                              // output rows retired (all items)
    int64_t item = my_a;
    int ye = 0, y = 0, i = 0, r0 = 0, r1 = 0, nend = 0, nnext = 0;
    uint32_t lofs = 0;                            // byte offset of this lane's 12 bytes inside a staged row
    uint32_t gstride = kRowB;                     // row stride of a whole staging group (pitch when one bulk copy)
    const int* y1 = nullptr;
    auto open = [&]() {                           // item `item`: its band's source rows, window ends, footprint
      const TItem t = decode_item<NV, NH * PPL, kBand>(vx, cnt, item, plans, p);
      const vp_clip_plan& pl = plans[t.k];
      int j0, jn, pa, np;
      slice_span(pl, t.ws, t.s, j0, jn, pa, np);
      y1 = y1tab + (int64_t)tab_alias[t.k] * kTabOutStride;
      const int o = (3 * pa) & 15;
      lofs = (uint32_t)(o + 384 * warp + 12 * lane);   // the footprint starts at (3*pa) & 15
      const int64_t pit = pitch_arr[t.k];
      gstride = pit == (int64_t)((o + 3 * np + 15) & ~15) ? (uint32_t)pit : (uint32_t)kRowB;   // as issue_group
      r0 = t.r0;
      r1 = t.r1;
      if (!kBand) {
        y = 0;
        ye = pl.in_h;
        i = 0;
        nend = __ldg(y1);
        nnext = __ldg(y1 + 1);
        return;
      }
      y = band_ys(pl, r0);
      ye = __ldg(y1 + r1 - 1);
      // rows above the band still live at its first source row are accumulated and dropped (never stored): the
      // ring slot of row r0-q is that of row r0+4-q, which starts only after row r0-q ended (<= 4 live rows)
      i = r0;
      while (i > 0 && __ldg(y1 + i - 1) > y) --i;
      nend = __ldg(y1 + i);
      nnext = __ldg(y1 + i + 1);
      const float2 z2 = make_float2(0.f, 0.f);   // band items leave partial rows below r1 in the ring
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          h2(acc[r][q], 0) = __fmul2_rn(h2(acc[r][q], 0), z2);
          h2(acc[r][q], 1) = __fmul2_rn(h2(acc[r][q], 1), z2);
        }
    };
    // clear a ring slot as a[q] * 0 (6 FMUL2; the accumulators are finite): ptxas materialises literal zeros here as
    // 18 uniform-register moves
    auto clear = [&](float4 (&a)[3]) {
      const float2 z2 = make_float2(0.f, 0.f);
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        h2(a[q], 0) = __fmul2_rn(h2(a[q], 0), z2);
        h2(a[q], 1) = __fmul2_rn(h2(a[q], 1), z2);
      }
    };
    // retire output row i (ring slot C = i % 4) into retire slot rr % kNR.  Preset geometry (kStatic: every out_h is
    // a multiple of 4, so rr % 4 == i % 4): the retire slot is C itself and its addresses are immediates.  A row
    // above the item's band (keep = false) is only cleared.
    auto retire = [&](float4 (&a)[3], auto cslot, bool keep) {
      constexpr int C = decltype(cslot)::value;
      const uint32_t rs = kStatic ? (uint32_t)C : rr % kNR;
      if (keep) {
        mbar_wait_uni<VP_TEAM_HINT>(&rempty[rs], ((rr / kNR) & 1) ^ 1);
        const uint32_t so_ = rs * kSlotB;
        sts_f4(vo[0] + so_, a[0]);               // pixels 0..2 are quads .xyz; pixel 3 is the .w column
        sts_f4(vo[1] + so_, a[1]);
        sts_f4(vo[2] + so_, a[2]);
        sts_f4(vo[3] + so_, make_float4(a[0].w, a[1].w, a[2].w, 0.f));
      }
      clear(a);
      if (keep) {
        __syncwarp();
        mbar_arrive_if(&rfull[rs], l0 || VP_ALL_LANES_ARRIVE);
        ++rr;
      }
    };
    // one staged row (converted): FMA into the ring (static slots), retire the output rows it completes
    auto fma_row = [&](const float2 (&fv)[6], const float4 wv) {
      const float ws[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const float2 ww = make_float2(ws[s], ws[s]);
#pragma unroll
        for (int c = 0; c < 6; ++c) h2(acc[s][c >> 1], c & 1) = __ffma2_rn(ww, fv[c], h2(acc[s][c >> 1], c & 1));
      }
      ++y;
      while (y == nend) {                         // source row y-1 completed output row i (ring slot i % 4)
        const bool keep = !kBand || i >= r0;
        switch (i & 3) {
          case 0: retire(acc[0], std::integral_constant<int, 0>{}, keep); break;
          case 1: retire(acc[1], std::integral_constant<int, 1>{}, keep); break;
          case 2: retire(acc[2], std::integral_constant<int, 2>{}, keep); break;
          default: retire(acc[3], std::integral_constant<int, 3>{}, keep); break;
        }
        ++i;
        nend = !kBand || i < r1 ? nnext : 0x7fffffff;   // the band (or the sentinels past out_h) ends the chain
        nnext = __ldg(y1 + i + 1);
      }
    };
    auto row = [&](uint32_t n0, uint32_t n1, uint32_t n2, float4 wv) {
      float2 fv[6];
      cvt_ring(n0, n1, n2, fv);
      fma_row(fv, wv);
    };
    open();
    // fresh: this group starts an item, so the producer filled it row by row (issue_group opens items inside its
    // per-row path): walk it with the per-row addressing
    bool fresh = true;
    for (;;) {
      if (y == ye) {                              // item done (all its output rows retired)
        if (++item >= my_b) break;
        open();
        fresh = true;
      }
      const uint32_t g = (rc / kTGrp) % kTNGrp;
      const uint32_t par = (rc / kTDepth) & 1;
      mbar_wait_uni(&sfull[g], par);
      const uint32_t gst = stage_s + g * (kTGrp * kRowB);
      const uint32_t gw = wrec_s + g * (kTGrp * 16);
      bool fin = false;
      if (!fresh && ye - y >= kTGrp) {
        // the whole group belongs to this item: rows in pairs with two register sets, each row's bytes loaded one
        // row and converted half a row ahead of its FMAs (the conversions of row q+1 overlap the FMAs of row q in
        // one basic block); the look-ahead past the group wraps to its own consumed rows (no stray reads).
        const uint32_t sb = gst + lofs;
        auto ld3 = [&](int r, uint32_t& x0, uint32_t& x1, uint32_t& x2) {
          const uint32_t sa = sb + (uint32_t)r * gstride;
          x0 = lds_u32(sa); x1 = lds_u32(sa + 4); x2 = lds_u32(sa + 8);
        };
        uint32_t ra0, ra1, ra2, rb0, rb1, rb2;
        float2 fa[6], fb[6];
        ld3(0, ra0, ra1, ra2);
        float4 wa = lds_f4(gw);
        ld3(1, rb0, rb1, rb2);
        float4 wb = lds_f4(gw + 16);
        cvt_ring(ra0, ra1, ra2, fa);
#pragma unroll 1
        for (int q = 0; q < kTGrp; q += 2) {
          const int q2 = (q + 2) & (kTGrp - 1), q3 = (q + 3) & (kTGrp - 1);
          cvt_ring(rb0, rb1, rb2, fb);
          ld3(q2, ra0, ra1, ra2);
          fma_row(fa, wa);
          wa = lds_f4(gw + q2 * 16);
          cvt_ring(ra0, ra1, ra2, fa);
          ld3(q3, rb0, rb1, rb2);
          fma_row(fb, wb);
          wb = lds_f4(gw + q3 * 16);
        }
      } else {
        // the group straddles items (or ends the CTA's range)
#pragma unroll 1
        for (int q = 0; q < kTGrp; ++q) {
          if (y == ye) {
            if (++item >= my_b) { fin = true; break; }
            open();
          }
          const uint32_t sa = gst + lofs + q * kRowB;
          row(lds_u32(sa), lds_u32(sa + 4), lds_u32(sa + 8), lds_f4(gw + q * 16));
        }
      }
      if (fin) break;
      fresh = false;
      rc += kTGrp;
      // the last V warp to finish group g refills it
      if (VP_ALL_LANES_ARRIVE) mbar_arrive(&sread[g]);
      __syncwarp();
      int old = 0;
      if (l0) {
        __threadfence_block();
        old = atomicAdd(&gcnt[g], 1);
        if (old == NV - 1) gcnt[g] = 0;
      }
      if (__shfl_sync(0xffffffffu, old, 0) == NV - 1) {
        if (VP_ALL_LANES_ARRIVE) mbar_wait_uni(&sread[g], par);
        issue_group(g);
      }
    }
    return;
  }

  // =================================================================== H warps
  const int hw = warp - NV;
  const int B = m * p, D = 3 * tp * p * p;
  const int cstride = tp * p * p;                 // elements between channel blocks of a patch row (O8)
  constexpr int kEsz = kF32 ? 4 : 2;
  int cur_j = -1, cur_s = -1;
  float2 wp[PPL][kUL];                            // pair weights per union tap
  uint32_t toff[PPL][kUL];                        // shared addresses of the taps in retire slot 0
  int colpart[PPL];
  bool hact[PPL];
  uint32_t rr = 0;
  for (int64_t item = my_a; item < my_b; ++item) {
    const TItem t = decode_item<NV, NH * PPL, kBand>(vx, cnt, item, plans, p);
    const vp_clip_plan& pl = plans[t.k];
    if (hw == 0 && l0 && tab_flag[tab_alias[t.k]] != 0 && clip_status != nullptr) clip_status[t.k] = VP_EUNSUPPORTED;
    if (t.j != cur_j || t.s != cur_s) {
      // ---- K2 for this slice: union window of each of my column pairs, f64 Keys / f64 sums -> fp32 ----
      cur_j = t.j;
      cur_s = t.s;
      int j0, jn, pa, np;
      slice_span(pl, t.ws, t.s, j0, jn, pa, np);
#pragma unroll
      for (int pp = 0; pp < PPL; ++pp) {
        const int q = pp * NH * 32 + hw * 32 + lane;
        hact[pp] = 2 * q < jn;
        const int ja = j0 + 2 * min(q, max(jn / 2 - 1, 0));
        const Win w0 = window_of(pl.in_w, pl.out_w, ja);
        const Win w1 = window_of(pl.in_w, pl.out_w, ja + 1);
        double s0 = 0.0, s1 = 0.0;
        for (int x = w0.x0; x < w0.x1; ++x) s0 += keys_d(((double)x - w0.c + 0.5) * w0.inv);
        for (int x = w1.x0; x < w1.x1; ++x) s1 += keys_d(((double)x - w1.c + 0.5) * w1.inv);
        const double r0 = s0 != 0.0 ? s0 : 1.0, r1 = s1 != 0.0 ? s1 : 1.0;
        const int xu = min(w0.x0, w1.x0);
        if (hact[pp] && max(w0.x1, w1.x1) - xu > kUL && clip_status != nullptr) clip_status[t.k] = VP_EUNSUPPORTED;
        // rotated tap order (see rpos): lane's tap tt reads row position xu - pa + u with u = (tt - (xu - pa)) mod UL,
        // so at every tap all lanes read positions of one residue class mod UL -- distinct banks under rpos
        const int rot = !kLarge ? (kUL - (xu - pa) % kUL) % kUL : 0;
#pragma unroll
        for (int tt = 0; tt < kUL; ++tt) {
          const int u = tt + rot < kUL ? tt + rot : tt + rot - kUL;
          const int x = xu + u;
          const float wa = (x >= w0.x0 && x < w0.x1) ? (float)(keys_d(((double)x - w0.c + 0.5) * w0.inv) / r0) : 0.f;
          const float wb = (x >= w1.x0 && x < w1.x1) ? (float)(keys_d(((double)x - w1.c + 0.5) * w1.inv) / r1) : 0.f;
          wp[pp][tt] = kFold ? make_float2(wa * kp.scale[0], wb * kp.scale[0]) : make_float2(wa, wb);
          toff[pp][tt] = kLarge ? buf_s + (uint32_t)(xu - pa + u) * 16u        // padded row: base + 16 u
                                : buf_s + (uint32_t)pos(min(x - pa, kPx - 1)) * 16u;   // slack taps (weight 0) stay in the row
        }
        const int jl0 = ja % B, wbk = ja / B, mw = jl0 / p, px = jl0 - mw * p;
        colpart[pp] = (wbk * m * m + mw) * D + px;
      }
    }
    // ---- output addressing of frame f (O7, O8): element (row, q) of pixel_values at row*D + q ----
    void* pv = pl.is_image ? pv_img : pv_vid;
    const int64_t cap = pl.is_image ? img_cap : vid_cap;
    const bool writable = pv != nullptr && pl.patch_offset + (int64_t)pl.grid_t * pl.grid_h * pl.grid_w <= cap;
    const int f = t.f;
    const int last_slot = (f == pl.n_frames - 1) ? pl.grid_t * tp - 1 : f;     // frame n-1 fills the pad slots
    const int nslots = last_slot - f + 1;
    const int g0 = f / tp, ti0 = f - g0 * tp;
    const int64_t group_stride = (int64_t)(pl.grid_h / m) * (pl.grid_w / m) * m * m * D;
    const int hb_stride = (pl.grid_w / m) * m * m * D;        // one merge-row band of one temporal group
    char* const fbase = reinterpret_cast<char*>(pv) +
        (pl.patch_offset * (int64_t)D + (int64_t)g0 * group_stride + (int64_t)ti0 * p * p) * kEsz;
    bool hst[PPL];
#pragma unroll
    for (int pp = 0; pp < PPL; ++pp) hst[pp] = writable && hact[pp];
    auto hrow = [&](uint32_t so, char* const (&qb)[PPL]) {   // H of one retired row in slot offset so
#pragma unroll
      for (int pp = 0; pp < PPL; ++pp) {
        if (hst[pp]) {
          float2 ar, ag, ab;
          if (kFold) {
            ar = make_float2(kp.bias[0], kp.bias[0]);
            ag = make_float2(kp.bias[1], kp.bias[1]);
            ab = make_float2(kp.bias[2], kp.bias[2]);
          } else {
            ar = ag = ab = make_float2(0.f, 0.f);
          }
#pragma unroll
          for (int u = 0; u < kUL; ++u) {
            const float4 v = lds_f4(toff[pp][u] + so);
            ar = __ffma2_rn(make_float2(v.x, v.x), wp[pp][u], ar);
            ag = __ffma2_rn(make_float2(v.y, v.y), wp[pp][u], ag);
            ab = __ffma2_rn(make_float2(v.z, v.z), wp[pp][u], ab);
          }
          store_pair<kF32, kFold>(kp, qb[pp], ar, ag, ab, cstride, nslots, ti0, tp, p, group_stride);
        }
      }
    };
    if (kStatic) {
      for (int ib = t.r0; ib < t.r1; ib += 4) {
        // row offset of output row i (O8): (i / (m p)) * hb_stride + ((i / p) % m) * m * D + (i % p) * p; the 4 rows
        // of a group share i / p
        const int ro_grp = (ib / B) * hb_stride + ((ib / p) % m) * m * D + (ib % p) * p;
        const uint32_t par = (rr / kNR) & 1;
        const uint32_t sbase = kNR == 4 ? 0u : ((rr >> 2) % (uint32_t)(kNR / 4)) * 4u;
        char* gb[PPL];                              // output address of row ib, per column pair
#pragma unroll
        for (int pp = 0; pp < PPL; ++pp) gb[pp] = fbase + (int64_t)(ro_grp + colpart[pp]) * kEsz;
#pragma unroll
        for (int U = 0; U < 4; ++U) {
          char* qb[PPL];
#pragma unroll
          for (int pp = 0; pp < PPL; ++pp) qb[pp] = gb[pp] + U * p * kEsz;   // rows ib..ib+3 share i / p
          mbar_wait_uni<VP_TEAM_HINT>(&rfull[sbase + U], par);
          hrow((sbase + (uint32_t)U) * kSlotB, qb);
          __syncwarp();
          mbar_arrive_if(&rempty[sbase + U], l0 || VP_ALL_LANES_ARRIVE);
        }
        rr += 4;
      }
    } else {
      for (int i = t.r0; i < t.r1; ++i) {
        const uint32_t rs = rr % kNR;
        mbar_wait_uni<VP_TEAM_HINT>(&rfull[rs], (rr / kNR) & 1);
        char* qb[PPL];
#pragma unroll
        for (int pp = 0; pp < PPL; ++pp)
          qb[pp] = fbase + (int64_t)((i / B) * hb_stride + ((i / p) % m) * m * D + (i % p) * p + colpart[pp]) * kEsz;
        hrow(rs * kSlotB, qb);
        __syncwarp();
        mbar_arrive_if(&rempty[rs], l0 || VP_ALL_LANES_ARRIVE);
        ++rr;
      }
    }
  }
}


// ---------------------------------------------------------------- per-clip vertical tables (K2 for KV_TEAM)
// y1tab[j][i] = end of output row i's window (then 4 sentinels 0x7fffffff); vtab[j][y] = fp32 weights
// (f64 Keys / f64 window sum, C10) of the output rows i(y)..i(y)+3 in ring-slot order (row r at r % 4), i(y) = first
// output row with y1 > y: the row the kernel is completing when it consumes source row y.  One table per run of equal (in_h, out_h) in the list.
__device__ __forceinline__ double win_sum(const Win& w) {
  double s = 0.0;
  for (int x = w.x0; x < w.x1; ++x) s += keys_d(((double)x - w.c + 0.5) * w.inv);
  return s;
}

__device__ __forceinline__ bool teamish(const vp_clip_plan& pl, int64_t coff, int64_t pitch) {
  return pl.status == VP_OK && pl.tile_count > 0 &&
         (pl.kernel_variant == KV_TEAM || pl.kernel_variant == KV_WIDE || pl.kernel_variant == KV_TEAML) &&
         ((coff | pitch) & 15) == 0;
}

__global__ void __launch_bounds__(128)
team_vtab_kernel(const vp_clip_plan* __restrict__ plans, const int64_t* __restrict__ coff,
                 const int64_t* __restrict__ pitch, const int* __restrict__ alias, float4* __restrict__ vtab,
                 int* __restrict__ y1tab, int* __restrict__ tflag) {
  const int j = blockIdx.y;                       // clip index (tables are indexed by the run's first clip)
  const vp_clip_plan& pl = plans[j];
  if (!teamish(pl, coff[j], pitch[j]) || alias[j] != j) return;
  const int in_h = pl.in_h, out_h = pl.out_h;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < out_h + 4) y1tab[(int64_t)j * kTabOutStride + r] = r < out_h ? window_of(in_h, out_h, r).x1 : 0x7fffffff;
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
    if (q < 4) wv[(i + q) & 3] = (float)wt;       // slot order: output row i + q lives in ring slot (i + q) % 4
    else if (fabs(wt) > 1e-9) atomicOr(&tflag[j], 1);     // a 5th live row with a non-negligible weight
  }
  vtab[(int64_t)j * kTabInH + y] = make_float4(wv[0], wv[1], wv[2], wv[3]);
}

// ---------------------------------------------------------------- per-variant work index
// One CTA: slot v in {MILD, MEDIUM, STRONG, COPY, TEAM, WIDE} collects the valid, 16-B aligned clips of that
// variant (list, batch order) and the exclusive prefix of their item counts (off); meta[v] = {count, items}.  For
// the TEAM / WIDE clips, alias[k] = first clip of the run of consecutive such clips with equal (in_h, out_h) that k
// belongs to: the clips of a run share one vertical table.
constexpr int kIdxThreads = 1024;
__device__ __forceinline__ int variant_slot(int kv) {
  return kv == KV_COPY ? 3 : (kv == KV_TEAM ? 4 : (kv == KV_WIDE ? 5 : (kv == KV_TEAML ? 6 : (kv == KV_U8 ? 7 : (kv <= KV_STRONG ? kv : -1)))));
}

__global__ void __launch_bounds__(kIdxThreads)
variant_index_kernel(const vp_clip_plan* __restrict__ plans, int n, const int64_t* __restrict__ coff,
                     const int64_t* __restrict__ pitch, int* __restrict__ list, int64_t* __restrict__ off,
                     int64_t* __restrict__ meta, int* __restrict__ alias, int* __restrict__ tflag, int num_sms) {
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
      // TMA variants need 16-B aligned rows; the u8 kernel reads bytes and takes any alignment
      if (pl.status == VP_OK && pl.tile_count > 0 &&
          (pl.kernel_variant == KV_U8 || ((coff[k] | pitch[k]) & 15) == 0)) {
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
  if (tid < kNSlots) off[(size_t)tid * (n + 1) + c_cnt[tid]] = c_items[tid];
  // ---- row bands for the team slots (TEAM, WIDE, TEAML) of launches with too few items to fill the GPU ----
  __shared__ unsigned long long tb[3][kMaxBands];
  __shared__ int s_nb[kNSlots];
  if (tid < 3 * kMaxBands) tb[tid / kMaxBands][tid % kMaxBands] = 0ull;
  if (tid < kNSlots) s_nb[tid] = 1;
  __syncthreads();
  for (int v = 4; v <= 6; ++v) {
    const int cn = c_cnt[v];
    // only launches with fewer than 4 items per CTA are candidates (large launches skip the band sums)
    if ((double)c_items[v] >= 4.0 * num_sms * (v == 5 ? 1 : 2)) continue;
    for (int c0 = 0; c0 < cn; c0 += kIdxThreads) {
      const int q = c0 + tid;
      const vp_clip_plan* pl = q < cn ? &plans[list[(size_t)v * n + q]] : nullptr;
#pragma unroll 1
      for (int nb = 1; nb <= kMaxBands; ++nb) {
        unsigned long long x = pl ? (unsigned long long)pl->tile_count * band_count(pl->out_h, nb) : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0 && x) atomicAdd(&tb[v - 4][nb - 1], x);
      }
    }
  }
  __syncthreads();
  if (tid < 3) {
    // CTAs of the launch: KV_WIDE one per SM, KV_TEAM / KV_TEAML two; score = busy fraction of the last wave,
    // discounted 3% per extra band (halo rows, per-item setup); large launches keep whole frames
    const int v = 4 + tid;
    const double G = (double)num_sms * (v == 5 ? 1 : 2);
    int best = 1;
    if ((double)tb[tid][0] < 4.0 * G && tb[tid][0] > 0) {
      double bs = -1.0;
      for (int nb = 1; nb <= kMaxBands; ++nb) {
        const double per = (double)tb[tid][nb - 1] / G;
        const double eff = per < 1.0 ? per : per / ceil(per);
        const double sc = eff / (1.0 + 0.03 * (nb - 1));
        if (sc > bs + 1e-9) { bs = sc; best = nb; }
      }
    }
    s_nb[v] = best;
  }
  __syncthreads();
  for (int v = 4; v <= 6; ++v) {
    const int nb = s_nb[v];
    if (nb == 1) continue;
    // rebuild the slot's item prefix with tile_count x bands per clip (block scan over its list)
    int64_t carry = 0;
    const int cn = c_cnt[v];
    for (int c0 = 0; c0 < cn; c0 += kIdxThreads) {
      const int q = c0 + tid;
      int64_t x = 0;
      if (q < cn) {
        const vp_clip_plan& pl = plans[list[(size_t)v * n + q]];
        x = (int64_t)pl.tile_count * band_count(pl.out_h, nb);
      }
      int64_t inc = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
      }
      if (lane == 31) wsum[warp][0] = inc;
      __syncthreads();
      int64_t pre = carry, tot = 0;
      for (int w = 0; w < kIdxThreads / 32; ++w) {
        if (w < warp) pre += wsum[w][0];
        tot += wsum[w][0];
      }
      if (q < cn) off[(size_t)v * (n + 1) + q] = pre + inc - x;
      __syncthreads();
      carry += tot;
    }
    if (tid == 0) {
      off[(size_t)v * (n + 1) + cn] = carry;
      c_items[v] = carry;
    }
    __syncthreads();
  }
  if (tid < kNSlots) {
    meta[4 * tid] = c_cnt[tid];
    meta[4 * tid + 1] = c_items[tid];
    meta[4 * tid + 2] = s_nb[tid];
    meta[4 * tid + 3] = 0;
  }
  __syncthreads();
  // table aliases: inclusive max-scan of run starts over the clips
  for (int c0 = 0; c0 < n; c0 += kIdxThreads) {
    const int k = c0 + tid;
    int v = -1;
    if (k < n) {
      tflag[k] = 0;
      const vp_clip_plan& a = plans[k];
      if (teamish(a, coff[k], pitch[k])) {
        bool start = k == 0;
        if (!start) {
          const vp_clip_plan& b = plans[k - 1];
          start = !teamish(b, coff[k - 1], pitch[k - 1]) || a.in_h != b.in_h || a.out_h != b.out_h;
        }
        v = start ? k : -1;
      }
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) v = max(v, __shfl_up_sync(0xffffffffu, v, o));
    if (lane == 31) wmax[warp] = v;
    __syncthreads();
    int pre = c_alias;
    for (int w = 0; w < warp; ++w) pre = max(pre, wmax[w]);
    if (k < n) alias[k] = max(pre, v);
    __syncthreads();
    if (tid == kIdxThreads - 1) c_alias = max(pre, v);
    __syncthreads();
  }
}

// Per-device SM-count cache (thread-safe: idempotent writes).
constexpr int kMaxDev = 64;
std::atomic<int> g_sms[kMaxDev];

// Dynamic shared memory above 48 KB must be opted into per kernel and device; cudaFuncSetAttribute is a cheap
// host-side call and idempotent, so it is simply made before every launch (no process state to get wrong when
// one process drives several devices or host threads).
template <typename K>
void set_smem_attr(K kern, int, int bytes) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

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
  const size_t o_meta = take(4 * kNSlots * sizeof(int64_t));
  const size_t o_alias = take((size_t)n * sizeof(int));
  const size_t o_flag = take((size_t)n * sizeof(int));
  const size_t o_vtab = take((size_t)n * kTabInH * sizeof(float4));
  const size_t o_y1 = take((size_t)n * kTabOutStride * sizeof(int));
  const size_t o_u8 = take((size_t)n * sizeof(int2));
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
    w.u8prec = reinterpret_cast<int2*>(b + o_u8);
  }
  return w;
}

VIdx ws_vidx(const ResizeWs& w, int n, int slot) {
  return VIdx{w.list + (size_t)slot * n, w.off + (size_t)slot * (n + 1), w.meta + 4 * slot};
}

cudaError_t launch_index(const vp_clip_plan* plans, int n, const int64_t* coff, const int64_t* pitch,
                         const ResizeWs& w, int num_sms, cudaStream_t s) {
  variant_index_kernel<<<1, kIdxThreads, 0, s>>>(plans, n, coff, pitch, w.list, w.off, w.meta, w.alias, w.tflag,
                                                   num_sms);
  return cudaGetLastError();
}

template <int NV, int NH, int PPL, int MINB, bool kF32, int kUL = kTeamUL, bool kLarge = false>
void launch_split(const FKParams& kp, bool preset, const vp_clip_plan* plans, const VIdx& vx, const ResizeWs& w,
                  const uint8_t* frames, const int64_t* coff, const int64_t* pitch, void* pi, int64_t icap, void* pvv,
                  int64_t vcap, int32_t* clip_status, int dev, int num_sms, cudaStream_t s) {
  using Cfg = SplitCfg<NV, NH, kLarge>;
  // Qwen2.5/3-VL geometry (p16 m2 tp2) with compile-time output addressing, else runtime parameters
  // a channel-uniform scale (e.g. Qwen mean = std = 0.5) folds into the horizontal weights (store_pair)
  const bool fold = kp.scale[0] == kp.scale[1] && kp.scale[1] == kp.scale[2];
  auto pick = [&](auto band) {
    constexpr bool B = decltype(band)::value;
    return preset ? (fold ? resize_split_kernel<NV, NH, PPL, kUL, kF32, true, 16, 2, 2, MINB, kLarge, B>
                          : resize_split_kernel<NV, NH, PPL, kUL, kF32, false, 16, 2, 2, MINB, kLarge, B>)
                  : resize_split_kernel<NV, NH, PPL, kUL, kF32, false, 0, 0, 0, MINB, kLarge, B>;
  };
  // whole-frame and row-band instantiations: the device-side band choice (meta[2]) lets exactly one of them run
  auto launch = [&](auto kern) {
    set_smem_attr(kern, dev, (int)Cfg::SMEM);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, Cfg::kThreads, Cfg::SMEM);
    if (per_sm < 1) per_sm = 1;
    kern<<<num_sms * per_sm, Cfg::kThreads, Cfg::SMEM, s>>>(kp, plans, vx, w.alias, w.tflag, w.vtab, w.y1tab, frames,
                                                            coff, pitch, pi, icap, pvv, vcap, clip_status);
  };
  launch(pick(std::false_type{}));
  launch(pick(std::true_type{}));
}

cudaError_t launch_team(const FKParams& kp, const vp_clip_plan* plans, int n, const ResizeWs& w, const uint8_t* frames,
                        const int64_t* coff, const int64_t* pitch, void* pi, int64_t icap, void* pvv, int64_t vcap,
                        int32_t* clip_status, int dev, int num_sms, unsigned mask, cudaStream_t s) {
  dim3 tg((kTabInH + 127) / 128, n);   // kTabInH >= kTabOutStride
  team_vtab_kernel<<<tg, 128, 0, s>>>(plans, coff, pitch, w.alias, w.vtab, w.y1tab, w.tflag);
  const bool preset = kp.p == 16 && kp.m == 2 && kp.tp == 2;
  const bool team = (mask >> KV_TEAM) & 1u, wide = (mask >> KV_WIDE) & 1u, large = (mask >> KV_TEAML) & 1u;
  if (large) {
    if (kp.out_f32)
      launch_split<kTeamNV, kTeamNH, 1, 2, true, kTeamULL, true>(kp, preset, plans, ws_vidx(w, n, 6), w, frames, coff,
                                                                pitch, pi, icap, pvv, vcap, clip_status, dev, num_sms, s);
    else
      launch_split<kTeamNV, kTeamNH, 1, 2, false, kTeamULL, true>(kp, preset, plans, ws_vidx(w, n, 6), w, frames, coff,
                                                                 pitch, pi, icap, pvv, vcap, clip_status, dev, num_sms, s);
  }
  if (kp.out_f32) {
    if (team)
      launch_split<kTeamNV, kTeamNH, kTeamPPL, 2, true>(kp, preset, plans, ws_vidx(w, n, 4), w, frames, coff, pitch, pi,
                                                        icap, pvv, vcap, clip_status, dev, num_sms, s);
    if (wide)
      launch_split<kWideNV, kWideNH, kWidePPL, 1, true>(kp, preset, plans, ws_vidx(w, n, 5), w, frames, coff, pitch, pi,
                                                        icap, pvv, vcap, clip_status, dev, num_sms, s);
  } else {
    if (team)
      launch_split<kTeamNV, kTeamNH, kTeamPPL, 2, false>(kp, preset, plans, ws_vidx(w, n, 4), w, frames, coff, pitch, pi,
                                                         icap, pvv, vcap, clip_status, dev, num_sms, s);
    if (wide)
      launch_split<kWideNV, kWideNH, kWidePPL, 1, false>(kp, preset, plans, ws_vidx(w, n, 5), w, frames, coff, pitch, pi,
                                                         icap, pvv, vcap, clip_status, dev, num_sms, s);
  }
  return cudaGetLastError();
}

}  // namespace vp
