// vp_resize_fast.cu -- K3 fast path: streaming fused AA-bicubic resize + clamp + normalise +
// temporal pad + patchify (O4-O9) for the common ratios (KV_MILD / KV_MEDIUM / KV_STRONG).
//
// Work item = (clip, source frame f, strip of Ws <= 256 output columns).  A CTA walks the item's
// source rows top to bottom exactly once with two warp-specialised groups:
//   * 4 V warps (vertical pass).  Each V warp owns a 128-pixel (384-byte) slice of the strip's
//     source footprint and keeps kDepth (16) rows of it in flight with cp.async.bulk (global -> smem,
//     refilled in groups of 8, completion on per-group mbarriers); the producer state is warp-uniform and only the copy /
//     barrier instructions are predicated to lane 0.  Lane L converts its 4 pixels (12 bytes) once per
//     source row (I2F.U8 on the XU pipe for 2 of its 3 words, PRMT into 2^23 + b and FADD2 -2^23 for the
//     third: both exact) and FMAs them (FFMA2, broadcast weight) into
//     the output rows live at that row, held in a register ring acc[5] of float4 quads.  Output row i
//     lives in slot i % 5; the output-row loop is unrolled by 5 so every slot index is static (no
//     dynamic register indexing, no accumulator shuffles).
//   * 4 H warps (horizontal pass).  Retired rows arrive through a 4-row smem buffer in row pairs
//     (mbarrier hand-off each way), pixel-major float4 (RGB + pad) in a sub-pixel-major layout inside
//     32-pixel blocks (vpos: conflict-free V stores, 1.35x H read wavefronts).  Each H thread computes a
//     column pair x 2 rows x 3 channels over the pair's union window (LDS.128 per tap and row, 3 FFMA2:
//     the pixel broadcast against the pair's weights), normalises, clamps in the output domain and
//     stores bf16x2 / float2 straight into the HF patch layout, once per temporal slot the frame fills
//     (O7) -- every output element is written exactly once.
// Registers are rebalanced between the warpgroups with setmaxnreg (V 152: the 60-register ring; H 104).
// Per-clip tables (cached across a CTA's consecutive items): per source row the fp32 weights (f64 Keys /
// f64 window sum) of its live output rows; windows are trimmed of exact-zero taps (identity axes become
// 1-tap copies).  Per item: the strip's horizontal weights.  Measurements behind each choice: DESIGN.md
// section 6 and profiles/r03_summary.md.
#include "vp_k3_common.cuh"
#include <atomic>

// setmaxnreg split between the V and H warpgroups (sum 256): V needs its 152 registers
constexpr int kVRegs = 152, kHRegs = 104;
#ifndef VP_ALL_LANES_ARRIVE
#define VP_ALL_LANES_ARRIVE 0   // verification build only (scripts/sanitize.sh): every lane arrives on vfull/vempty
#endif

namespace vp {
namespace {

constexpr int kNVW = 4;                   // V warps
constexpr int kNHW = 4;                   // H warps
constexpr int kNT = (kNVW + kNHW) * 32;   // 256 threads
// Staging depth / refill group / V->H buffer rows.  16/8/4 measured 3% faster than 8/4/6 on cfg5: the refill
// (ProdState round trip, expect_tx, address setup) is paid once per 8 rows instead of 4, and the smem for the
// deeper ring comes from the V->H buffer (its depth is irrelevant above 2 row pairs).
#ifndef VP_DEPTH
#define VP_DEPTH 16
#endif
#ifndef VP_GRP
#define VP_GRP 8
#endif
#ifndef VP_CAPR
#define VP_CAPR 4
#endif
constexpr int kDepth = VP_DEPTH;          // source rows in flight per V warp (refilled in groups of kGrp)
static_assert((kDepth & (kDepth - 1)) == 0, "the staging position is a masked running counter");
constexpr int kGrp = VP_GRP;              // rows per TMA group (one mbarrier phase per group)
constexpr int kNGrp = kDepth / kGrp;
constexpr int kWarpPx = 128;              // pixels per V warp slice (32 lanes x 4 px)
constexpr int kWarpB = 3 * kWarpPx;       // 384 bytes
constexpr int kCapR = VP_CAPR;            // retired-row buffer rows (V -> H), in row pairs
constexpr int kRowPx = kFastPx;           // float4 pixels per buffered row (union-slack taps wrap, weight 0)


// Footprint of a strip: first pixel (16-aligned so that the byte offset 3*pa is 16-B aligned for TMA)
// and pixel count.
struct Strip {
  int j0, jn, pa, np;
};
__device__ __forceinline__ Strip strip_of(const vp_clip_plan& pl, int ws, int strip) {
  Strip s;
  s.j0 = strip * ws;
  s.jn = min(ws, pl.out_w - s.j0);
  s.pa = window_of(pl.in_w, pl.out_w, s.j0).x0 & ~15;
  s.np = window_of(pl.in_w, pl.out_w, s.j0 + s.jn - 1).x1 - s.pa;
  return s;
}


// ---------------------------------------------------------------- vertical ring
// acc[slot].q[j]: this lane's 12 source bytes (4 RGB pixels: R0 G0 B0 R1 | G1 B1 R2 G2 | B2 R3 G3 B3) for the
// output row in `slot`, as three float4 quads -- bytes (2q, 2q+1) are the .xy / .zw halves (FFMA2 operands)
// and pixels 0 and 2 are whole quads at retire (no repacking).
struct AccRow {
  float4 q[3];
};
typedef AccRow Acc[kRing];

__device__ __forceinline__ float2& half2_of(float4& v, int h) { return reinterpret_cast<float2*>(&v)[h]; }

// contributions of one source row to the live rows i..i+4, where row i sits in slot U (static).
// Dense over the ring slots: the weight vector holds 0 for rows that are not live, so the code is
// straight-line FFMA2 with no per-row branch (a 0-weight FMA adds exactly 0).
template <int U>
__device__ __forceinline__ void ring_row(Acc& acc, const float (&w)[kRing], const float2 (&f)[6]) {
#pragma unroll
  for (int r = 0; r < kRing; ++r) {
    const int slot = (U + r) % kRing;
    const float2 ww = make_float2(w[r], w[r]);
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      float2& a = half2_of(acc[slot].q[q >> 1], q & 1);
      a = __ffma2_rn(ww, f[q], a);
    }
  }
}

// Retired-row layout: footprint pixel x (float4 RGB + pad) sits at float4 index vpos(x): inside each block of
// 32 pixels, sub-pixel-major (pixel 4a + k at 8k + a).  The V lanes' retire stores (pixels 4L + k, lane L)
// then hit 8 distinct 16-B granules per quarter-warp (conflict-free), and the H lanes' tap reads (column
// pairs ~2*scale pixels apart) cost 1.35 wavefronts per ideal one at the cfg2 ratio (natural layout 2.9,
// an XOR swizzle 1.95; offline bank simulation over the tap pattern).
__device__ __forceinline__ int vpos(int x) {
  x &= kRowPx - 1;                  // union-slack taps past the footprint (zero weight) wrap to finite data
  return (x & ~31) | ((x & 3) << 3) | ((x & 31) >> 2);
}
// byte offset of footprint pixel x inside a retired row (pixel-major float4 at vpos(x))
__device__ __forceinline__ int hoff(int x) {
  return vpos(x) * (int)sizeof(float4);
}

// store the finished output row of slot S as 4 pixel-major float4 (R, G, B, pad) at this lane's pixel
// positions (row + vb + 8k: vpos of pixel 4L + k inside the 32-px block layout) and clear the slot.  The pad
// of pixels 0 and 2 is whatever the quad holds (H reads .xyz only).
template <int S>
__device__ __forceinline__ void retire_slot(Acc& acc, float4* __restrict__ row, int vb, bool active) {
  if (active) {
    const float4* a = acc[S].q;
    row[vb] = a[0];                                            // R0 G0 B0 (R1)
    row[vb + 8] = make_float4(a[0].w, a[1].x, a[1].y, 0.f);    // R1 G1 B1
    row[vb + 16] = make_float4(a[1].z, a[1].w, a[2].x, a[2].y); // R2 G2 B2 (R3)
    row[vb + 24] = make_float4(a[2].y, a[2].z, a[2].w, 0.f);   // R3 G3 B3
  }
#pragma unroll
  for (int j = 0; j < 3; ++j) acc[S].q[j] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// 4 bytes of w -> two float2 pairs (b0,b1), (b2,b3): PRMT builds the float 2^23 + b (exact), FADD2 removes
// 2^23.  ALU + FMA pipes instead of I2F.U8 (16/clk/SM on B200, measured: scripts/ubench.cu).
__device__ __forceinline__ void bytes_to_f2_i2f(uint32_t w, float2& lo, float2& hi) {   // XU pipe (I2F.U8)
  lo = make_float2((float)(w & 0xffu), (float)((w >> 8) & 0xffu));
  hi = make_float2((float)((w >> 16) & 0xffu), (float)(w >> 24));
}
__device__ __forceinline__ void bytes_to_f2(uint32_t w, float2& lo, float2& hi) {
  const float2 mm = make_float2(-8388608.f, -8388608.f);
  lo = __fadd2_rn(make_float2(__uint_as_float(__byte_perm(w, 0x4B000000u, 0x7540u)),
                              __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7541u))), mm);
  hi = __fadd2_rn(make_float2(__uint_as_float(__byte_perm(w, 0x4B000000u, 0x7542u)),
                              __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7543u))), mm);
}


template <bool kF32>
__device__ __forceinline__ void store_slots(void* pv, int64_t idx, float v0, float v1, int nslots, int ti0, int tp,
                                            int p, int64_t group_stride) {
  for (int s2 = 0, ti = ti0; s2 < nslots; ++s2) {
    if (kF32) *reinterpret_cast<float2*>(reinterpret_cast<float*>(pv) + idx) = make_float2(v0, v1);
    else *reinterpret_cast<__nv_bfloat162*>(reinterpret_cast<__nv_bfloat16*>(pv) + idx) = __floats2bfloat162_rn(v0, v1);
    if (++ti == tp) { ti = 0; idx += group_stride - (int64_t)(tp - 1) * p * p; }
    else idx += (int64_t)p * p;
  }
}

// ---------------------------------------------------------------- configuration per variant
template <int VARIANT>
struct FastCfg {
  // union of two adjacent columns' windows: LHM + the largest start shift between them (<= ceil(fs)+1)
  static constexpr int UL = VARIANT == KV_MILD ? 11 : (VARIANT == KV_MEDIUM ? 23 : 51);
  static constexpr int MAXWS = kFastMaxWs;
  static constexpr size_t OFF_STG = 0;                                                   // V staging
  static constexpr size_t OFF_VBUF = OFF_STG + (size_t)kNVW * kDepth * kWarpB;          // retired rows
  static constexpr size_t OFF_WROW = OFF_VBUF + (size_t)kCapR * kRowPx * 16;   // float4 [kInHMax] + float [kInHMax]
  static constexpr size_t OFF_Y1 = OFF_WROW + (size_t)kInHMax * 20;
  static constexpr size_t OFF_WH = OFF_Y1 + (size_t)kOutHMax * 4;
  static constexpr size_t OFF_HX = OFF_WH + (size_t)kWhFloats * 4;
  static constexpr size_t OFF_BAR = (OFF_HX + (size_t)MAXWS * 4 + 15) & ~(size_t)15;
  static constexpr size_t OFF_PROD = OFF_BAR + (kNVW * kNGrp + 2 * (kCapR / 2)) * 8;   // ProdState [kNVW]
  static constexpr size_t OFF_EBAR = OFF_PROD + (size_t)kNVW * 32;                      // verification build only
  static constexpr size_t SMEM = OFF_EBAR + (size_t)kNVW * kNGrp * 8;
  static_assert(OFF_VBUF % 16 == 0 && OFF_WROW % 16 == 0 && OFF_WH % 16 == 0, "align");
  static_assert(SMEM + 1024 <= 228 * 1024 / 2, "two CTAs per SM");
};

// Per-V-warp TMA producer (lane 0): walks the CTA's item sequence and keeps its slice of kDepth rows
// in flight.  issue() refills the slot of the row the warp has just finished reading.  The per-item
// setup is a separate non-inlined function returning by value, so the per-row state stays in registers.
// TMA producer state of one V warp, kept in shared memory (read/written once per 4-row refill) so that it
// does not occupy registers in the register-bound V loop.
struct ProdState {
  const uint8_t* src;   // next source row of the slice
  int64_t pitch;
  int64_t next;         // next item to open
  int rows, nbytes;     // rows left in the current item, bytes per row of the slice
};
static_assert(sizeof(ProdState) == 32, "ProdState");

struct ProdItem {
  const uint8_t* src;   // this warp's slice of source row 0 of the item (nullptr: no more items)
  int64_t pitch;
  int64_t item;         // item index of this slice
  int in_h, nbytes;
};

template <int VARIANT>
__device__ __forceinline__ ProdItem producer_open(const vp_clip_plan* __restrict__ plans, const VIdx vx, int cnt, int w,
                                               const uint8_t* __restrict__ frames,
                                               const int64_t* __restrict__ clip_off,
                                               const int64_t* __restrict__ pitch_arr, int64_t item, int64_t my_b) {
  ProdItem r;
  r.src = nullptr;
  r.pitch = 0;
  r.item = item;
  r.in_h = 0;
  r.nbytes = 0;
  if (item < my_b) {
    const int j = vfind(vx, cnt, item);
    const int k = vx.list[j];
    const vp_clip_plan pl = plans[k];
    const int64_t coff = clip_off[k], pitch = pitch_arr[k];
    const int ws = fast_strip_width(pl.in_w, pl.out_w);
    const int nstrips = (pl.out_w + ws - 1) / ws;
    const int64_t local = item - vx.off[j];
    const int f = (int)(local / nstrips), strip = (int)(local % nstrips);
    const Strip st = strip_of(pl, ws, strip);
    const int px0 = st.pa + w * kWarpPx;                       // this warp's first pixel
    const int pxn = min(kWarpPx, st.pa + st.np - px0);         // its pixels (may be <= 0)
    // 16-B multiple, never past the 16-B rounded row end (pitch is a multiple of 16 >= 3*in_w)
    r.nbytes = pxn > 0 ? min(kWarpB, (3 * (px0 + pxn) + 15) / 16 * 16 - 3 * px0) : 0;
    r.src = frames + coff + (int64_t)f * pl.in_h * pitch + 3 * (int64_t)px0;
    r.pitch = pitch;
    r.in_h = pl.in_h;
    r.item = item;
    return r;
  }
  r.item = item;
  return r;
}

template <int VARIANT, bool kF32>
__global__ void __launch_bounds__(kNT, 2)
resize_fast_kernel(FKParams kp, const vp_clip_plan* __restrict__ plans, const VIdx vx, const uint8_t* __restrict__ frames,
                   const int64_t* __restrict__ clip_off, const int64_t* __restrict__ pitch_arr, void* pv_img,
                   int64_t img_cap, void* pv_vid, int64_t vid_cap) {
  using Cfg = FastCfg<VARIANT>;
  constexpr int UL = Cfg::UL;
  extern __shared__ __align__(128) unsigned char smem[];
  uint8_t* stage_all = smem + Cfg::OFF_STG;
  float4* vbuf = reinterpret_cast<float4*>(smem + Cfg::OFF_VBUF);
  // vertical weights per source row: w[0..3] (float4) and w[4] of its live output rows i0..i0+4
  float4* w4t = reinterpret_cast<float4*>(smem + Cfg::OFF_WROW);
  float* w1t = reinterpret_cast<float*>(smem + Cfg::OFF_WROW + (size_t)kInHMax * 16);
  int* y1t = reinterpret_cast<int*>(smem + Cfg::OFF_Y1);
  float* wh = reinterpret_cast<float*>(smem + Cfg::OFF_WH);
  int* hx = reinterpret_cast<int*>(smem + Cfg::OFF_HX);
  uint64_t* full_all = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);   // [kNVW][kDepth]
  uint64_t* vfull = full_all + kNVW * kNGrp;                                // retired row pairs: V -> H
  uint64_t* ebar_all = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_EBAR);  // [kNVW][kNGrp] (VP_ALL_LANES_ARRIVE)
  uint64_t* vempty = vfull + kCapR / 2;                                     // H -> V

  const int tid = threadIdx.x;
  // warp index as a warp-uniform value and lane id from the special register (kept in registers, not
  // re-derived from %tid inside the row loops)
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  int lane;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(lane));

  // contiguous slice of this variant's items
  const int cnt = (int)vx.meta[0];
  const int64_t total = vx.meta[1];
  const int64_t my_a = total * blockIdx.x / gridDim.x;
  const int64_t my_b = total * (blockIdx.x + 1) / gridDim.x;

  if (tid == 0) {
    for (int s = 0; s < kNVW * kNGrp; ++s) {
      mbar_init(&full_all[s], 1);
      mbar_init(&ebar_all[s], 32);
    }
    for (int s = 0; s < kCapR / 2; ++s) {
      mbar_init(&vfull[s], 2 * kNVW * (VP_ALL_LANES_ARRIVE ? 32 : 1));   // each V warp arrives once per row of the pair
      mbar_init(&vempty[s], kNHW * (VP_ALL_LANES_ARRIVE ? 32 : 1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < kCapR * kRowPx; i += kNT) vbuf[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  __syncthreads();

  if (warp < kNVW) {
    // ============================================================ V warps: vertical ring
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" :: "n"(kVRegs) : "memory");
    uint8_t* stage = stage_all + (size_t)warp * kDepth * kWarpB;
    uint64_t* full = full_all + warp * kNGrp;     // one barrier per group of kGrp staging slots
    uint64_t* ebar = ebar_all + warp * kNGrp;     // verification build: the warp's reads of a group are done
    uint32_t rc = 0;                  // staged rows read so far: slot rc % kDepth, phase (rc / kDepth) & 1
    uint32_t vslot = 0, vphase = 0;   // vbuf slot of the next retired row and its pair phase (kCapR even:
                                      // vslot & 1 is the row's parity within its pair)
    int cached_clip = -1;
    // TMA producer: warp-uniform state (every lane tracks it), copies / barrier ops predicated to lane 0,
    // so the refill is not a divergent branch.  A group of kGrp rows inside one item is one expect_tx.
    const bool l0 = lane == 0;
    ProdState* ps = reinterpret_cast<ProdState*>(smem + Cfg::OFF_PROD) + warp;
    if (l0) *ps = ProdState{nullptr, 0, my_a, 0, 0};
    __syncwarp();
    // verification build (compute-sanitizer racecheck): every lane arrives on ebar[g] after reading group g and
    // waits for the phase before the TMA refill (the shipped kernel relies on the __syncwarp before the refill)
    auto reads_done = [&](uint32_t g, uint32_t parity) {
      if (VP_ALL_LANES_ARRIVE) {
        mbar_arrive(&ebar[g]);
        mbar_wait(&ebar[g], parity);
      }
    };
    auto issue_group = [&](uint32_t g) {          // refill the kGrp slots of group g, then arrive once
      // opaque copy of g (nvcc 12.9 CSE workaround, see vp_resize_ring.cu)
      asm volatile("mov.b32 %0, %0;" : "+r"(g));
      ProdState st = *ps;                         // warp-uniform (broadcast smem reads)
      if (st.rows >= kGrp) {
        mbar_expect_tx_if(&full[g], (uint32_t)(kGrp * st.nbytes), l0);
#pragma unroll
        for (int q = 0; q < kGrp; ++q)
          tma_bulk_g2s_if(stage + (size_t)(g * kGrp + q) * kWarpB, st.src + (int64_t)q * st.pitch,
                          (uint32_t)st.nbytes, &full[g], l0 && st.nbytes > 0);
        st.src += (int64_t)kGrp * st.pitch;
        st.rows -= kGrp;
      } else {
#pragma unroll 1
        for (int q = 0; q < kGrp; ++q) {
          if (st.rows == 0 && st.next < my_b) {
            const ProdItem pit =
                producer_open<VARIANT>(plans, vx, cnt, warp, frames, clip_off, pitch_arr, st.next, my_b);
            ++st.next;
            st.src = pit.src;
            st.pitch = pit.pitch;
            st.rows = pit.in_h;
            st.nbytes = pit.nbytes;
          }
          if (st.rows > 0) {
            mbar_expect_tx_if(&full[g], (uint32_t)st.nbytes, l0);
            tma_bulk_g2s_if(stage + (size_t)(g * kGrp + q) * kWarpB, st.src, (uint32_t)st.nbytes, &full[g],
                            l0 && st.nbytes > 0);
            st.src += st.pitch;
            --st.rows;
          }
        }
      }
      mbar_arrive_if(&full[g], l0);
      __syncwarp();                               // every lane has read *ps
      if (l0) *ps = st;
      __syncwarp();
    };
    for (uint32_t g = 0; g < kNGrp; ++g) issue_group(g);     // prefill
    int64_t item = my_a;
    while (item < my_b) {
      const int j = vfind(vx, cnt, item);
      const int k = vx.list[j];
      const vp_clip_plan pl = plans[k];
      const int64_t cbase = vx.off[j], cend = vx.off[j + 1];
      const int ws = fast_strip_width(pl.in_w, pl.out_w);
      const int nstrips = (pl.out_w + ws - 1) / ws;
      const int in_h = pl.in_h, out_h = pl.out_h;
      if (k != cached_clip) {
        // ---- vertical tables for this clip (K2), V warps only: y1 per output row; per source row y the
        //      weights of its live rows i0..i0+4 (relative order; 0 where not live), f64 Keys / window sum ----
        named_sync(1, kNVW * 32);
        for (int i = tid; i < out_h; i += kNVW * 32) y1t[i] = window_of(in_h, out_h, i).x1;
        named_sync(1, kNVW * 32);
        const double sc = (double)in_h / (double)out_h;
        const double sup = 2.0 * (sc > 1.0 ? sc : 1.0);
        for (int y = tid; y < in_h; y += kNVW * 32) {
          int i = (int)floor(((double)y - sup - 0.5) / sc - 0.5);
          if (i < 0) i = 0;
          if (i > out_h) i = out_h;
          while (i > 0 && y1t[i - 1] > y) --i;
          while (i < out_h && y1t[i] <= y) ++i;
          float wv[kRing] = {0.f, 0.f, 0.f, 0.f, 0.f};
          for (int r = 0; r < kRing && i + r < out_h; ++r) {
            const Win w = window_of(in_h, out_h, i + r);
            if (w.x0 > y) break;
            double s = 0.0;
            for (int yy = w.x0; yy < w.x1; ++yy) s += keys_d(((double)yy - w.c + 0.5) * w.inv);
            wv[r] = (float)(keys_d(((double)y - w.c + 0.5) * w.inv) / (s != 0.0 ? s : 1.0));
          }
          w4t[y] = make_float4(wv[0], wv[1], wv[2], wv[3]);
          w1t[y] = wv[4];
        }
        named_sync(1, kNVW * 32);
        cached_clip = k;
      }
      // this clip's items in the slice as 32-bit local indices (fewer live 64-bit values in the row loop)
      const int l_end = (int)((cend < my_b ? cend : my_b) - cbase);
      for (int local = (int)(item - cbase); local < l_end; ++local) {
        const Strip st = strip_of(pl, ws, local % nstrips);
        const int px_lane = warp * kWarpPx + lane * 4;      // this lane's first pixel (relative to pa)
        const bool vactive = px_lane < st.np;
        // vpos(px_lane + k) == vb + 8k for this lane's 4 pixels (px_lane is a multiple of 4)
        const int vb = vpos(px_lane);
        Acc acc;
#pragma unroll
        for (int r = 0; r < kRing; ++r)
#pragma unroll
          for (int j = 0; j < 3; ++j) acc[r].q[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        int y = 0;
        // No software prefetch: with 16 warps per SM the LDS latency of a row is covered by other warps, and
        // loading at the top of the row keeps the loop free of register rotation copies (measured faster).
        uint32_t n0 = 0, n1 = 0, n2 = 0;
        auto load_bytes = [&]() {
          if ((rc & (kGrp - 1)) == 0) mbar_wait(&full[(rc / kGrp) % kNGrp], (rc / kDepth) & 1);   // per group
          const uint32_t* sp = reinterpret_cast<const uint32_t*>(stage + (rc % kDepth) * kWarpB) + lane * 3;
          n0 = sp[0]; n1 = sp[1]; n2 = sp[2];
        };

        // Output row i lives in ring slot i % kRing.  Unrolling the output-row loop by kRing makes every
        // slot index static: for row i = ib + U, consume the source rows up to its window end y1_i (the
        // first live row of each of them is i), then retire slot U.
        for (int ib = 0; ib < out_h; ib += kRing) {
          int yends[kRing];                        // window ends of rows ib..ib+4, loaded once per group
#pragma unroll
          for (int u = 0; u < kRing; ++u) yends[u] = y1t[min(ib + u, out_h - 1)];
#define VP_ROW(U)                                                                               \
          if (ib + U < out_h) {                                                                 \
            const int yend = yends[U];                                                          \
            for (; y < yend; ++y) {                                                             \
              load_bytes();                                                                     \
              const float4 wa = w4t[y];                                                         \
              const float wb = w1t[y];                                                          \
              float2 fv[6];                   /* bytes (2q, 2q+1) as exact floats (PRMT + FADD2) */ \
              bytes_to_f2_i2f(n0, fv[0], fv[1]);   /* 2 of 3 words on the XU pipe (I2F.U8) */   \
              bytes_to_f2_i2f(n1, fv[2], fv[3]);                                                \
              bytes_to_f2(n2, fv[4], fv[5]);       /* 1 on ALU + FMA (PRMT + FADD2) */          \
              const uint32_t used = rc++ % kDepth;                                              \
              if ((used & (kGrp - 1)) == kGrp - 1) {   /* group read: refill it */                \
                __syncwarp();                                                                   \
                reads_done(used / kGrp, ((rc - 1) / kDepth) & 1);                               \
                issue_group(used / kGrp);                                                       \
              }                                                                                 \
              const float w5[kRing] = {wa.x, wa.y, wa.z, wa.w, wb};                             \
              ring_row<U>(acc, w5, fv);                                                         \
            }                                                                                   \
            const uint32_t vs = vslot, vp2 = vs >> 1, vph = vphase;                             \
            if ((vs & 1) == 0) mbar_wait(&vempty[vp2], vph ^ 1);    /* per pair */              \
            retire_slot<U>(acc, vbuf + vs * kRowPx, vb, vactive);                               \
            __syncwarp();                                                                       \
            if (lane == 0 || VP_ALL_LANES_ARRIVE) mbar_arrive(&vfull[vp2]);                                            \
            if (++vslot == kCapR) { vslot = 0; vphase ^= 1; }                                   \
          }
          static_assert(kRing == 5, "unroll below");
          VP_ROW(0) VP_ROW(1) VP_ROW(2) VP_ROW(3) VP_ROW(4)
#undef VP_ROW
        }
        if (vslot & 1) {                            // odd out_h: complete the last pair's barrier phase
          __syncwarp();
          if (lane == 0 || VP_ALL_LANES_ARRIVE) mbar_arrive(&vfull[vslot >> 1]);
          if (++vslot == kCapR) { vslot = 0; vphase ^= 1; }
        }
        // source rows below the last window (none for the supported ratios) keep the ring in step
        for (; y < in_h; ++y) {
          if ((rc & (kGrp - 1)) == 0) mbar_wait(&full[(rc / kGrp) % kNGrp], (rc / kDepth) & 1);
          __syncwarp();
          const uint32_t used = rc++ % kDepth;
          if ((used & (kGrp - 1)) == kGrp - 1) {
            __syncwarp();
            reads_done(used / kGrp, ((rc - 1) / kDepth) & 1);
            issue_group(used / kGrp);
          }
        }
      }
      item = cbase + l_end;
    }
    return;
  }

  // ============================================================ H warps: horizontal pass + store
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" :: "n"(kHRegs) : "memory");
  const int ht = tid - kNVW * 32;       // 0..127
  const int p = kp.p, m = kp.m, tp = kp.tp, B = m * p;
  uint32_t vrow = 0;
  int64_t item = my_a;
  while (item < my_b) {
    const int j = vfind(vx, cnt, item);
    const int k = vx.list[j];
    const vp_clip_plan pl = plans[k];
    const int64_t cbase = vx.off[j], cend = vx.off[j + 1];
    void* pv = pl.is_image ? pv_img : pv_vid;
    const int64_t cap = pl.is_image ? img_cap : vid_cap;
    const bool writable = pv != nullptr && pl.patch_offset + (int64_t)pl.grid_t * pl.grid_h * pl.grid_w <= cap;
    const int ws = fast_strip_width(pl.in_w, pl.out_w);
    const int nstrips = (pl.out_w + ws - 1) / ws;
    const int out_h = pl.out_h;
    for (; item < cend && item < my_b; ++item) {
      const int64_t local = item - cbase;
      const int f = (int)(local / nstrips);
      const Strip st = strip_of(pl, ws, (int)(local % nstrips));
      // ---- horizontal weights of this strip: per column pair (ja, ja+1) the union of the two windows
      //      starting at x0(ja), UL taps, layout [pair][u][2] (0 outside each column's window) ----
      named_sync(2, kNHW * 32);
      for (int cpi = ht; cpi < (st.jn >> 1); cpi += kNHW * 32) {
        const Win w0 = window_of(pl.in_w, pl.out_w, st.j0 + 2 * cpi);
        const Win w1 = window_of(pl.in_w, pl.out_w, st.j0 + 2 * cpi + 1);
        double s0 = 0.0, s1 = 0.0;
        for (int x = w0.x0; x < w0.x1; ++x) s0 += keys_d(((double)x - w0.c + 0.5) * w0.inv);
        for (int x = w1.x0; x < w1.x1; ++x) s1 += keys_d(((double)x - w1.c + 0.5) * w1.inv);
        const double r0 = s0 != 0.0 ? 1.0 / s0 : 1.0, r1 = s1 != 0.0 ? 1.0 / s1 : 1.0;
        for (int u = 0; u < UL; ++u) {
          const int x = w0.x0 + u;
          wh[(cpi * UL + u) * 2] = (x < w0.x1) ? (float)(keys_d(((double)x - w0.c + 0.5) * w0.inv) * r0) : 0.f;
          wh[(cpi * UL + u) * 2 + 1] =
              (x >= w1.x0 && x < w1.x1) ? (float)(keys_d(((double)x - w1.c + 0.5) * w1.inv) * r1) : 0.f;
        }
        hx[cpi] = w0.x0 - st.pa;                      // union start relative to the footprint start
      }
      named_sync(2, kNHW * 32);
      const int npairs = st.jn >> 1;                 // jn is even (multiple of the even factor p*m)
      const bool hact = ht < npairs;
      const int ja = 2 * ht;
      const int xu = hact ? hx[ht] : 0;
      // swizzled float4 indices of this lane's taps (kept in registers for the MILD union)
      constexpr int kOffRegs = UL <= 11 ? UL : 1;
      int toff[kOffRegs];
#pragma unroll
      for (int u = 0; u < kOffRegs; ++u) toff[u] = hoff(xu + u);   // byte offsets
      // column part of the output element index (O8): (wb*m^2 + mw)*D + px  (channel part added per c)
      int colpart;
      {
        const int j = st.j0 + ja, wbk = j / B, jl = j - wbk * B, mw = jl / p, px = jl - mw * p;
        colpart = (wbk * m * m + mw) * kp.D + px;
      }
      const int cstride = tp * p * p;
      const int last_slot = (f == pl.n_frames - 1) ? pl.grid_t * tp - 1 : f;   // O7: frame n-1 fills pads
      const int gh = pl.grid_h, gw = pl.grid_w;
      const int g0 = f / tp, ti0 = f - g0 * tp;
      const int64_t group_stride = (int64_t)(gh / m) * (gw / m) * m * m * kp.D;
      const int64_t base0 = pl.patch_offset * (int64_t)kp.D + (int64_t)g0 * group_stride + (int64_t)ti0 * p * p;
      const int nslots = last_slot - f + 1;
      const int64_t hb_stride = (int64_t)(gw / m) * m * m * kp.D;
      // element offset of the next row to emit (incl. this thread's column part), advanced per row:
      // + p inside a patch row block, + d_mh when py wraps (next merge row), + d_hb when mh wraps too
      // (32-bit offset from the frame's 64-bit base: one frame's patch block is < 2^31 elements)
      const int64_t rbase = base0 + colpart;
      int rp = 0, r_mh = 0, r_py = 0;
      const int d_mh = m * kp.D - (p - 1) * p;
      const int d_hb = (int)hb_stride - (m - 1) * m * kp.D - (p - 1) * p;
      auto advance_row = [&]() {
        if (++r_py == p) {
          r_py = 0;
          if (++r_mh == m) { r_mh = 0; rp += d_hb; } else rp += d_mh;
        } else {
          rp += p;
        }
      };

      for (int i = 0; i < out_h; i += 2) {
        const bool two = i + 1 < out_h;
        const uint32_t s0 = vrow % kCapR, s1 = s0 + 1, ph0 = (vrow / kCapR) & 1;   // rows of pair s0/2
        mbar_wait(&vfull[s0 >> 1], ph0);
        const int64_t rp0 = rbase + rp;
        advance_row();
        const int64_t rp1 = rbase + rp;
        if (two) advance_row();
        if (writable && hact) {
          // row bases (warp-uniform) + per-lane byte offsets: one LDS.128 [R + UR] per tap and row
          const char* v0 = reinterpret_cast<const char*>(vbuf + s0 * kRowPx);
          const char* v1 = reinterpret_cast<const char*>(vbuf + (two ? s1 : s0) * kRowPx);
          // accumulators per (channel, row) over the column pair (col a, col b): each tap is 3 FFMA2 per row,
          // the pixel's channel value broadcast against the pair's weights (w_a, w_b)
          float2 ar0 = make_float2(0.f, 0.f), ag0 = ar0, ab0 = ar0, ar1 = ar0, ag1 = ar0, ab1 = ar0;
          const float2* wr = reinterpret_cast<const float2*>(wh) + ht * UL;
#pragma unroll
          for (int u = 0; u < UL; ++u) {
            const float2 wp = wr[u];                           // (col a, col b) weights at pixel xu+u
            const int o = UL <= 11 ? toff[u < kOffRegs ? u : 0] : hoff(xu + u);
            const float4 q0 = *reinterpret_cast<const float4*>(v0 + o);   // rows i, i+1 (.xyz = R, G, B)
            const float4 q1 = *reinterpret_cast<const float4*>(v1 + o);
            ar0 = __ffma2_rn(make_float2(q0.x, q0.x), wp, ar0);
            ag0 = __ffma2_rn(make_float2(q0.y, q0.y), wp, ag0);
            ab0 = __ffma2_rn(make_float2(q0.z, q0.z), wp, ab0);
            ar1 = __ffma2_rn(make_float2(q1.x, q1.x), wp, ar1);
            ag1 = __ffma2_rn(make_float2(q1.y, q1.y), wp, ag1);
            ab1 = __ffma2_rn(make_float2(q1.z, q1.z), wp, ab1);
          }
          // normalise (O6) x = v*scale_c + bias_c as FFMA2 over the column pair, then clamp (C12) in the
          // output domain: clamp(v,0,255)*s+b == clamp(v*s+b, b, 255*s+b) (s > 0), and for bf16
          // RNE(clamp(x)) == clamp(RNE(x), RNE(lo), RNE(hi)) (RNE is monotone) -> packed bf16x2 min/max.
          const float2 s0 = make_float2(kp.scale[0], kp.scale[0]), o0 = make_float2(kp.bias[0], kp.bias[0]);
          const float2 s1 = make_float2(kp.scale[1], kp.scale[1]), o1 = make_float2(kp.bias[1], kp.bias[1]);
          const float2 s2 = make_float2(kp.scale[2], kp.scale[2]), o2 = make_float2(kp.bias[2], kp.bias[2]);
          const float2 nr0 = __ffma2_rn(ar0, s0, o0);
          const float2 ng0 = __ffma2_rn(ag0, s1, o1);
          const float2 nb0 = __ffma2_rn(ab0, s2, o2);
          const float2 nr1 = __ffma2_rn(ar1, s0, o0);
          const float2 ng1 = __ffma2_rn(ag1, s1, o1);
          const float2 nb1 = __ffma2_rn(ab1, s2, o2);
          auto clampf2 = [&](float2 v, int c) {
            return make_float2(fminf(fmaxf(v.x, kp.lo[c]), kp.hi[c]), fminf(fmaxf(v.y, kp.lo[c]), kp.hi[c]));
          };
          auto packbf = [&](float2 v, int c) {
            const __nv_bfloat162 q = __floats2bfloat162_rn(v.x, v.y);
            return __hmin2(__hmax2(q, kp.lo2[c]), kp.hi2[c]);
          };
          const float2 xr0 = clampf2(nr0, 0), xg0 = clampf2(ng0, 1), xb0 = clampf2(nb0, 2);
          const float2 xr1 = clampf2(nr1, 0), xg1 = clampf2(ng1, 1), xb1 = clampf2(nb1, 2);
          const float xr0a = xr0.x, xr0b = xr0.y, xg0a = xg0.x, xg0b = xg0.y, xb0a = xb0.x, xb0b = xb0.y;
          const float xr1a = xr1.x, xr1b = xr1.y, xg1a = xg1.x, xg1b = xg1.y, xb1a = xb1.x, xb1b = xb1.y;
          if (nslots == 1) {
            // common case: one temporal slot -> 3 (or 6) stores at constant channel offsets from a row pointer
            if (kF32) {
              float* q0 = reinterpret_cast<float*>(pv) + rp0;
              *reinterpret_cast<float2*>(q0) = xr0;
              *reinterpret_cast<float2*>(q0 + cstride) = xg0;
              *reinterpret_cast<float2*>(q0 + 2 * cstride) = xb0;
              if (two) {
                float* q1 = reinterpret_cast<float*>(pv) + rp1;
                *reinterpret_cast<float2*>(q1) = xr1;
                *reinterpret_cast<float2*>(q1 + cstride) = xg1;
                *reinterpret_cast<float2*>(q1 + 2 * cstride) = xb1;
              }
            } else {
              __nv_bfloat16* q0 = reinterpret_cast<__nv_bfloat16*>(pv) + rp0;
              *reinterpret_cast<__nv_bfloat162*>(q0) = packbf(nr0, 0);
              *reinterpret_cast<__nv_bfloat162*>(q0 + cstride) = packbf(ng0, 1);
              *reinterpret_cast<__nv_bfloat162*>(q0 + 2 * cstride) = packbf(nb0, 2);
              if (two) {
                __nv_bfloat16* q1 = reinterpret_cast<__nv_bfloat16*>(pv) + rp1;
                *reinterpret_cast<__nv_bfloat162*>(q1) = packbf(nr1, 0);
                *reinterpret_cast<__nv_bfloat162*>(q1 + cstride) = packbf(ng1, 1);
                *reinterpret_cast<__nv_bfloat162*>(q1 + 2 * cstride) = packbf(nb1, 2);
              }
            }
          } else {
            // frame n-1 of a clip also fills the temporal pad slots (O7), images fill tp slots
            store_slots<kF32>(pv, rp0, xr0a, xr0b, nslots, ti0, tp, p, group_stride);
            store_slots<kF32>(pv, rp0 + cstride, xg0a, xg0b, nslots, ti0, tp, p, group_stride);
            store_slots<kF32>(pv, rp0 + 2 * cstride, xb0a, xb0b, nslots, ti0, tp, p, group_stride);
            if (two) {
              store_slots<kF32>(pv, rp1, xr1a, xr1b, nslots, ti0, tp, p, group_stride);
              store_slots<kF32>(pv, rp1 + cstride, xg1a, xg1b, nslots, ti0, tp, p, group_stride);
              store_slots<kF32>(pv, rp1 + 2 * cstride, xb1a, xb1b, nslots, ti0, tp, p, group_stride);
            }
          }
        }
        __syncwarp();
        if (lane == 0 || VP_ALL_LANES_ARRIVE) mbar_arrive(&vempty[s0 >> 1]);
        vrow += 2;                                  // V pads an odd last row, so pairs stay aligned
      }
    }
  }
}


// ---------------------------------------------------------------- KV_COPY (identity resize)
// Item = (clip, frame f, merge-row band hb, chunk wc of kCopyMW merge columns).  The band's B = m*p source
// rows x (<= kCopyMW*B) pixels are staged in shared memory with 16-B loads; each thread then owns fixed
// (channel, element-pair) positions of a patch's p x p chunk and walks the item's patches, writing
// bf16x2 / float2 pairs -- consecutive threads write consecutive elements of one chunk (coalesced).
// Numerics equal the fast kernel's on an identity axis pair (weights exactly 1): x*scale+bias, clamp
// in the output domain.
constexpr int kCT = 256;

template <bool kF32>
__global__ void __launch_bounds__(kCT)
resize_copy_kernel(FKParams kp, const vp_clip_plan* __restrict__ plans, const VIdx vx, const uint8_t* __restrict__ frames,
                   const int64_t* __restrict__ clip_off, const int64_t* __restrict__ pitch_arr, void* pv_img,
                   int64_t img_cap, void* pv_vid, int64_t vid_cap) {
  extern __shared__ __align__(16) unsigned char csm[];
  const int tid = threadIdx.x;
  const int p = kp.p, m = kp.m, tp = kp.tp, B = m * p, pp = p * p, half_pp = pp / 2;
  // contiguous slice of this variant's items
  const int cnt = (int)vx.meta[0];
  const int64_t total = vx.meta[1];
  const int64_t my_a = total * blockIdx.x / gridDim.x;
  const int64_t my_b = total * (blockIdx.x + 1) / gridDim.x;
  constexpr int kMaxW = 2;                          // element pairs per thread per pass over a patch
  const int npos = 3 * half_pp;                     // (channel, element pair) positions of one patch
  int64_t item = my_a;
  while (item < my_b) {
    const int j = vfind(vx, cnt, item);
    const int k = vx.list[j];
    const vp_clip_plan pl = plans[k];
    const int64_t cbase = vx.off[j], cend = vx.off[j + 1];
    const int64_t coff = clip_off[k], pitch = pitch_arr[k];
    void* pv = pl.is_image ? pv_img : pv_vid;
    const int64_t cap = pl.is_image ? img_cap : vid_cap;
    const bool writable = pv != nullptr && pl.patch_offset + (int64_t)pl.grid_t * pl.grid_h * pl.grid_w <= cap;
    const int gh = pl.grid_h, gw = pl.grid_w, nwc = copy_wchunks(gw, m), nhb = gh / m;
    const int64_t group_stride = (int64_t)nhb * (gw / m) * m * m * kp.D;
    for (; item < cend && item < my_b; ++item) {
      const int64_t local = item - cbase;
      const int f = (int)(local / ((int64_t)nhb * nwc));
      const int rem = (int)(local - (int64_t)f * nhb * nwc);
      const int hb = rem / nwc, wc = rem - hb * nwc;
      const int mc0 = wc * kCopyMW, nmc = min(kCopyMW, gw / m - mc0);   // merge columns of this item
      const int x0 = mc0 * B, ncols = nmc * B;
      const int rb = (3 * ncols + 15) & ~15;                           // staged row bytes (16-B multiple)
      const uint8_t* src = frames + coff + ((int64_t)f * pl.in_h + (int64_t)hb * B) * pitch + 3 * (int64_t)x0;
      __syncthreads();                                                 // previous item's readers are done
      const int q16 = rb >> 4;
      for (int i = tid; i < B * q16; i += kCT) {
        const int r = i / q16, q = i - r * q16;
        reinterpret_cast<uint4*>(csm + r * rb)[q] = __ldg(reinterpret_cast<const uint4*>(src + r * pitch) + q);
      }
      __syncthreads();
      if (!writable) continue;
      const int last_slot = (f == pl.n_frames - 1) ? pl.grid_t * tp - 1 : f;   // O7: frame n-1 fills pads
      const int nslots = last_slot - f + 1;
      const int g0 = f / tp, ti0 = f - g0 * tp;
      // patch row of (merge column mc, mh, mw) in slot group g0: patch_offset + ((g0*nhb + hb)*(gw/m) + mc)*m^2 + mh*m + mw
      const int64_t band_row = pl.patch_offset + ((int64_t)g0 * nhb + hb) * (gw / m) * m * m;
      const int npatch = nmc * m * m;
      for (int wb = 0; wb < npos; wb += kCT * kMaxW) {
        // this thread's fixed (channel, element pair) positions: w = c * pp/2 + e2
        int woff[kMaxW], wsrc[kMaxW];
        float wsc[kMaxW], wbi[kMaxW], wlo[kMaxW], whi[kMaxW];
        __nv_bfloat162 wlo2[kMaxW], whi2[kMaxW];
        bool wv[kMaxW];
#pragma unroll
        for (int t = 0; t < kMaxW; ++t) {
          const int w = wb + tid + t * kCT;
          wv[t] = w < npos;
          const int c = wv[t] ? w / half_pp : 0, e = wv[t] ? 2 * (w - c * half_pp) : 0;
          const int py = e / p, px = e - py * p;
          woff[t] = c * tp * pp + e + ti0 * pp;       // element offset inside the patch row (first slot)
          wsrc[t] = py * rb + 3 * px + c;             // staged byte offset inside the patch
          // per-channel constants selected without dynamic indexing of the parameter arrays
          wsc[t] = c == 0 ? kp.scale[0] : (c == 1 ? kp.scale[1] : kp.scale[2]);
          wbi[t] = c == 0 ? kp.bias[0] : (c == 1 ? kp.bias[1] : kp.bias[2]);
          wlo[t] = c == 0 ? kp.lo[0] : (c == 1 ? kp.lo[1] : kp.lo[2]);
          whi[t] = c == 0 ? kp.hi[0] : (c == 1 ? kp.hi[1] : kp.hi[2]);
          wlo2[t] = c == 0 ? kp.lo2[0] : (c == 1 ? kp.lo2[1] : kp.lo2[2]);
          whi2[t] = c == 0 ? kp.hi2[0] : (c == 1 ? kp.hi2[1] : kp.hi2[2]);
        }
        for (int pi = 0; pi < npatch; ++pi) {
          const int j = pi / (m * m), r2 = pi - j * m * m, mh = r2 / m, mw = r2 - mh * m;
          const int64_t prow = band_row + (int64_t)(mc0 + j) * m * m + r2;
          const uint8_t* sp = csm + (mh * p) * rb + 3 * (j * B + mw * p);
#pragma unroll
          for (int t = 0; t < kMaxW; ++t) {
            if (!wv[t]) continue;
            const uint8_t* s2 = sp + wsrc[t];
            const float v0 = fmaf((float)s2[0], wsc[t], wbi[t]);
            const float v1 = fmaf((float)s2[3], wsc[t], wbi[t]);
            int64_t idx = prow * kp.D + woff[t];
            if (kF32) {
              const float2 o = make_float2(fminf(fmaxf(v0, wlo[t]), whi[t]), fminf(fmaxf(v1, wlo[t]), whi[t]));
              for (int s2i = 0, ti = ti0; s2i < nslots; ++s2i) {
                *reinterpret_cast<float2*>(reinterpret_cast<float*>(pv) + idx) = o;
                if (++ti == tp) { ti = 0; idx += group_stride - (int64_t)(tp - 1) * pp; } else idx += pp;
              }
            } else {
              const __nv_bfloat162 o = __hmin2(__hmax2(__floats2bfloat162_rn(v0, v1), wlo2[t]), whi2[t]);
              for (int s2i = 0, ti = ti0; s2i < nslots; ++s2i) {
                *reinterpret_cast<__nv_bfloat162*>(reinterpret_cast<__nv_bfloat16*>(pv) + idx) = o;
                if (++ti == tp) { ti = 0; idx += group_stride - (int64_t)(tp - 1) * pp; } else idx += pp;
              }
            }
          }
        }
      }
    }
  }
}

// Per-device "attribute set" bits (thread-safe: cudaFuncSetAttribute is idempotent, the bits only skip repeats).
constexpr int kMaxDev = 64;
std::atomic<unsigned> g_attr_bits[kMaxDev];

template <typename K>
void ensure_smem_attr(K kern, int dev, unsigned bit, int bytes) {
  if (dev >= 0 && dev < kMaxDev && (g_attr_bits[dev].load(std::memory_order_acquire) & bit)) return;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (dev >= 0 && dev < kMaxDev) g_attr_bits[dev].fetch_or(bit, std::memory_order_acq_rel);
}

template <int VARIANT, bool kF32>
void launch_fast(const FKParams& kp, const vp_clip_plan* plans, const VIdx& vx, const uint8_t* frames,
                 const int64_t* coff, const int64_t* pitch, void* pi, int64_t icap, void* pvv, int64_t vcap,
                 int dev, int num_sms, cudaStream_t s) {
  using Cfg = FastCfg<VARIANT>;
  auto kern = resize_fast_kernel<VARIANT, kF32>;
  ensure_smem_attr(kern, dev, 1u << (2 * VARIANT + (kF32 ? 1 : 0)), (int)Cfg::SMEM);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kNT, Cfg::SMEM);
  if (per_sm < 1) per_sm = 1;
  kern<<<num_sms * per_sm, kNT, Cfg::SMEM, s>>>(kp, plans, vx, frames, coff, pitch, pi, icap, pvv, vcap);
}

template <bool kF32>
void launch_copy(const FKParams& kp, const vp_clip_plan* plans, const VIdx& vx, const uint8_t* frames,
                 const int64_t* coff, const int64_t* pitch, void* pi, int64_t icap, void* pvv, int64_t vcap,
                 int dev, int num_sms, cudaStream_t s) {
  auto kern = resize_copy_kernel<kF32>;
  const int B = kp.m * kp.p;
  const size_t smem = (size_t)B * ((3 * kCopyMW * B + 15) & ~15);
  ensure_smem_attr(kern, dev, 1u << (8 + (kF32 ? 1 : 0)), 200 * 1024);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kCT, smem);
  if (per_sm < 1) per_sm = 1;
  kern<<<num_sms * per_sm, kCT, smem, s>>>(kp, plans, vx, frames, coff, pitch, pi, icap, pvv, vcap);
}

}  // namespace

FKParams make_fkparams(const vp_params* p) {
  FKParams kp{};
  kp.p = p->patch_size;
  kp.m = p->merge_size;
  kp.tp = p->temporal_patch_size;
  kp.D = 3 * kp.tp * kp.p * kp.p;
  kp.out_f32 = p->out_dtype == VP_OUT_F32;
  for (int c = 0; c < 3; ++c) {
    kp.scale[c] = (float)(1.0 / (255.0 * p->std[c]));
    kp.bias[c] = (float)(-p->mean[c] / p->std[c]);
    // output-domain clamp bounds: the images of 0 and 255, ordered (std < 0 flips them)
    const float a = kp.bias[c], b = fmaf(255.0f, kp.scale[c], kp.bias[c]);
    kp.lo[c] = fminf(a, b);
    kp.hi[c] = fmaxf(a, b);
    kp.lo2[c] = __floats2bfloat162_rn(kp.lo[c], kp.lo[c]);
    kp.hi2[c] = __floats2bfloat162_rn(kp.hi[c], kp.hi[c]);
  }
  return kp;
}

// The warp-specialised streaming variants (MILD / MEDIUM / STRONG) and the identity copy, one launch each over
// that variant's items only (work index built by launch_index in the same workspace).
cudaError_t launch_fast_variants(const FKParams& kp, const vp_clip_plan* plans, int n, const ResizeWs& w,
                                 const uint8_t* frames, const int64_t* coff, const int64_t* pitch, void* pi,
                                 int64_t icap, void* pvv, int64_t vcap, int dev, int num_sms, unsigned mask,
                                 cudaStream_t s) {
  auto vx = [&](int slot) { return ws_vidx(w, n, slot); };
  auto has = [&](int kv) { return ((mask >> kv) & 1u) != 0; };
  if (kp.out_f32) {
    if (has(KV_MILD)) launch_fast<KV_MILD, true>(kp, plans, vx(0), frames, coff, pitch, pi, icap, pvv, vcap, dev, num_sms, s);
    if (has(KV_MEDIUM)) launch_fast<KV_MEDIUM, true>(kp, plans, vx(1), frames, coff, pitch, pi, icap, pvv, vcap, dev, num_sms, s);
    if (has(KV_STRONG)) launch_fast<KV_STRONG, true>(kp, plans, vx(2), frames, coff, pitch, pi, icap, pvv, vcap, dev, num_sms, s);
    if (has(KV_COPY)) launch_copy<true>(kp, plans, vx(3), frames, coff, pitch, pi, icap, pvv, vcap, dev, num_sms, s);
  } else {
    if (has(KV_MILD)) launch_fast<KV_MILD, false>(kp, plans, vx(0), frames, coff, pitch, pi, icap, pvv, vcap, dev, num_sms, s);
    if (has(KV_MEDIUM)) launch_fast<KV_MEDIUM, false>(kp, plans, vx(1), frames, coff, pitch, pi, icap, pvv, vcap, dev, num_sms, s);
    if (has(KV_STRONG)) launch_fast<KV_STRONG, false>(kp, plans, vx(2), frames, coff, pitch, pi, icap, pvv, vcap, dev, num_sms, s);
    if (has(KV_COPY)) launch_copy<false>(kp, plans, vx(3), frames, coff, pitch, pi, icap, pvv, vcap, dev, num_sms, s);
  }
  return cudaGetLastError();
}

}  // namespace vp
