// vp_resize_ring.cu -- K3 KV_RING: fused AA-bicubic resize + clamp + normalise + temporal pad + patchify
// (O4-O9, C10-C17) for clips whose two axes are downscales (or identity), one warp per CTA.
//
// Work item = (clip, strip of Ws output columns, source frame f), strip-major so that a CTA's consecutive
// items share the strip's horizontal table.  The warp streams the item's source rows top to bottom once:
//
//   V ring (lanes = 4 source pixels = 12 bytes each, 30 lanes = 120-pixel footprint).  Lane 0 keeps
//     kRDepth rows of the footprint in flight with cp.async.bulk (global -> smem, mbarrier complete_tx).
//     Each lane converts its 12 bytes once per row (PRMT into the float 2^23 + b, FADD2 -2^23: exact, and on
//     the ALU/FMA pipes instead of the 16/clk/SM I2F unit) and FMAs them (FFMA2, warp-uniform weight
//     broadcast) into the 5 ring slots; output row i lives in slot i % 5.  Every source row updates all 5
//     slots with weights stored in slot order (0 for rows not live), so the FMA code has no dependence on
//     which rows are live (at most 5 are, for a downscale).
//   Every kRHR = 20 output rows the warp switches to the H ring: lane (c, i) owns channel c of the rows i and
//     i + 10 of the block (a float2 pair); it walks the strip's footprint pixels left to right and FMAs each
//     pixel's pair (one LDS.64) into 5 column slots (column jj in slot jj % 5) with the pixel's warp-uniform
//     weights (slot order, FFMA2 broadcast).  When a column's window ends it is normalised, clamped (C12, in the
//     output domain), paired with its left neighbour into bf16x2 / float2 and staged in smem; when a
//     p-column block is complete the staged rows are written to the HF patch layout with 16-B stores
//     (every output element written once per temporal slot it fills, O7).
// Both loops are element-driven (one source row / pixel per iteration); the rows / columns whose windows end
// at an element retire after it (a 5-way switch on the slot; usually 0 or 1 per element).
// No other warp is involved, so there are no cross-warp barriers; 6 CTAs (warps) share an SM.
// Vertical weights come from a per-clip table in global memory (ring_vtables_kernel, L1-resident);
// horizontal weights are built per (clip, strip) in smem.  All weights: f64 Keys a = -0.5 -> fp32.
#include "vp_k3_common.cuh"

namespace vp {
namespace {

constexpr int kRT = 32;                 // one warp per CTA
constexpr int kRLanes = kRingPx / 4;    // 30 V lanes (4 px each)
constexpr int kRHR = 20;                // output rows per H block
constexpr int kRHP = kRHR / 2;          // H lanes = (channel, row pair (i, i + kRHP)): 3 x 10 = 30 lanes
constexpr int kRS = kRingPx + 1;        // pair-plane row stride in float2 (odd: conflict-free H reads)
constexpr int kRDepth = 8;              // staged source rows in flight
constexpr int kRGrp = 4;                // rows per TMA group barrier
constexpr int kRNGrp = kRDepth / kRGrp;
constexpr int kRStageB = 400;           // staged bytes per row: 3 * (kRingPx + 12 alignment px), 16-B multiple
static_assert(kRStageB >= 3 * (kRingPx + 12) && kRStageB % 16 == 0, "stage slot");
static_assert(kRHR % kRing == 0 && 3 * kRHP <= kRT, "H block");
constexpr size_t kVTabBytes = (size_t)24 * kRingInHMax;   // float4 w[0..3] + float w4 per source row, int y1 per output row

template <bool kF32>
struct RingCfg {
  // staged output row: 16 px; bf16 rows are 32 B with 8-B granules XOR-swizzled by (row >> 2) & 3 (<= 2-way
  // bank conflicts on the retire stores), f32 rows 64 B + 8 B pad
  static constexpr int OSTRIDE = kF32 ? 72 : 32;
  static constexpr size_t OFF_STG = 0;
  static constexpr size_t OFF_IP = OFF_STG + (size_t)kRDepth * kRStageB;                // float2 [3][kRHP][kRS]
  static constexpr size_t OFF_HW4 = (OFF_IP + (size_t)3 * kRHP * kRS * 8 + 15) & ~(size_t)15;   // float4 [kRS]
  static constexpr size_t OFF_HW2 = OFF_HW4 + (size_t)kRS * 16;                         // float2 [kRS]: (w4, pos)
  static constexpr size_t OFF_HX1 = OFF_HW2 + (size_t)kRS * 8;                          // int [kRingMaxWs + 1]
  static constexpr size_t OFF_RB = (OFF_HX1 + (size_t)(kRingMaxWs + 1) * 4 + 7) & ~(size_t)7;   // int64 [kRHR]
  static constexpr size_t OFF_OST = (OFF_RB + (size_t)kRHR * 8 + 15) & ~(size_t)15;     // [3][kRHR][OSTRIDE]
  static constexpr size_t OFF_BAR = (OFF_OST + (size_t)3 * kRHR * OSTRIDE + 7) & ~(size_t)7;
  static constexpr size_t SMEM = OFF_BAR + (size_t)kRNGrp * 8;
};

// Intermediate position of strip-local pixel q (lane q/4, sub-pixel q%4): sub-pixel-major so that the V
// lanes' retire stores are contiguous (conflict-free).
__device__ __forceinline__ int ipos(int q) { return (q & 3) * kRLanes + (q >> 2); }

struct VTab {
  const float4* w4;
  const float* w1;
  const int* y1;
};
__device__ __forceinline__ VTab vtab_at(const char* vt, int slot) {
  const char* b = vt + (size_t)slot * kVTabBytes;
  return VTab{reinterpret_cast<const float4*>(b), reinterpret_cast<const float*>(b + (size_t)16 * kRingInHMax),
              reinterpret_cast<const int*>(b + (size_t)20 * kRingInHMax)};
}

// byte k of w as the float 2^23 + byte (exact); the FADD2 of -2^23 follows in cvt12
__device__ __forceinline__ float magic_byte(uint32_t w, uint32_t k) {
  return __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7540u | k));
}

// 12 bytes (4 RGB pixels) -> (R,G) pairs of pixels 0..3 and (B0,B1), (B2,B3)
__device__ __forceinline__ void cvt12(uint32_t w0, uint32_t w1, uint32_t w2, float2 (&rg)[4], float2 (&b)[2]) {
  const float2 mm = make_float2(-8388608.f, -8388608.f);
  rg[0] = __fadd2_rn(make_float2(magic_byte(w0, 0), magic_byte(w0, 1)), mm);
  rg[1] = __fadd2_rn(make_float2(magic_byte(w0, 3), magic_byte(w1, 0)), mm);
  rg[2] = __fadd2_rn(make_float2(magic_byte(w1, 2), magic_byte(w1, 3)), mm);
  rg[3] = __fadd2_rn(make_float2(magic_byte(w2, 1), magic_byte(w2, 2)), mm);
  b[0] = __fadd2_rn(make_float2(magic_byte(w0, 2), magic_byte(w1, 1)), mm);
  b[1] = __fadd2_rn(make_float2(magic_byte(w2, 0), magic_byte(w2, 3)), mm);
}

struct VAcc {
  float2 rg[4];
  float2 b[2];
};

// Item decode: list position j, clip k, strip st, frame f.
struct RItem {
  int j, k, st, f;
};
__device__ __forceinline__ RItem ring_item(const vp_clip_plan* __restrict__ plans, const VIdx& vx, int cnt,
                                           int64_t item) {
  RItem r;
  r.j = vfind(vx, cnt, item);
  r.k = vx.list[r.j];
  const int64_t local = item - vx.off[r.j];
  const int nf = plans[r.k].n_frames;
  r.st = (int)(local / nf);
  r.f = (int)(local - (int64_t)r.st * nf);
  return r;
}

// first source pixel the V lanes cover for strip st: the first column's window start rounded down to 4 px
__device__ __forceinline__ int strip_pl(int in_w, int out_w, int j0) { return window_of(in_w, out_w, j0).x0 & ~3; }

// TMA producer (lane 0): source pointer / bytes / rows of the item it is staging.
struct RProd {
  const uint8_t* src;
  int64_t pitch;
  int64_t item;
  int rows, nbytes;
};

__device__ __forceinline__ RProd ring_prod_open(const vp_clip_plan* __restrict__ plans, const VIdx vx, int cnt,
                                             const uint8_t* __restrict__ frames, const int64_t* __restrict__ coff,
                                             const int64_t* __restrict__ pitch_arr, int64_t item, int64_t my_b) {
  RProd r{nullptr, 0, item, 0, 0};
  if (item >= my_b) return r;
  const RItem it = ring_item(plans, vx, cnt, item);
  const vp_clip_plan pl = plans[it.k];
  const int ws = ring_strip_width(pl.in_w, pl.out_w);
  const int pl0 = strip_pl(pl.in_w, pl.out_w, it.st * ws);
  const int pa = pl0 & ~15;                                  // 16-px aligned: 3*pa is a 16-B multiple
  const int rowend = (3 * pl.in_w + 15) & ~15;               // <= pitch (16-B multiple >= 3*in_w)
  r.nbytes = min(kRStageB, rowend - 3 * pa);
  r.pitch = pitch_arr[it.k];
  r.src = frames + coff[it.k] + (int64_t)it.f * pl.in_h * r.pitch + 3 * (int64_t)pa;
  r.rows = pl.in_h;
  return r;
}

template <bool kF32>
__global__ void __launch_bounds__(kRT, 6)
resize_ring_kernel(FKParams kp, const vp_clip_plan* __restrict__ plans, const VIdx vx,
                   const uint8_t* __restrict__ frames, const int64_t* __restrict__ clip_off,
                   const int64_t* __restrict__ pitch_arr, void* pv_img, int64_t img_cap, void* pv_vid, int64_t vid_cap,
                   const char* __restrict__ vt, const int* __restrict__ vt_owner) {
  using Cfg = RingCfg<kF32>;
  extern __shared__ __align__(128) unsigned char smem[];
  uint8_t* stage = smem + Cfg::OFF_STG;
  float* iP = reinterpret_cast<float*>(smem + Cfg::OFF_IP);        // [3][kRHP][kRS][2]
  float4* hw4 = reinterpret_cast<float4*>(smem + Cfg::OFF_HW4);
  float2* hw2 = reinterpret_cast<float2*>(smem + Cfg::OFF_HW2);
  int* hx1 = reinterpret_cast<int*>(smem + Cfg::OFF_HX1);
  int64_t* rbase = reinterpret_cast<int64_t*>(smem + Cfg::OFF_RB);
  unsigned char* ost = smem + Cfg::OFF_OST;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);

  int lane;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(lane));
  const int cnt = (int)vx.meta[0];
  const int64_t total = vx.meta[1];
  const int64_t my_a = total * blockIdx.x / gridDim.x;
  const int64_t my_b = total * (blockIdx.x + 1) / gridDim.x;
  if (my_a >= my_b) return;

  if (lane == 0) {
    for (int g = 0; g < kRNGrp; ++g) mbar_init(&bars[g], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  // ---- TMA producer: warp-uniform state; only the copies / barrier ops are predicated to lane 0 ----
  RProd pit{nullptr, 0, my_a, 0, 0};
  bool pstarted = false;
  const uint8_t* psrc = nullptr;
  int prows = 0;
  const bool l0 = lane == 0;
  // rows of group g (kRGrp staging slots), then one arrive on the group's barrier
  auto issue_group = [&](uint32_t g) {
    // Opaque copy of g: nvcc 12.9 otherwise CSEs &bars[g] with the wait path's barrier address computed
    // under the wait branch's condition, giving a misaligned barrier address here.
    asm volatile("mov.b32 %0, %0;" : "+r"(g));
#pragma unroll
    for (int q = 0; q < kRGrp; ++q) {
      if (prows == 0 && (!pstarted || pit.src != nullptr)) {
        pit = ring_prod_open(plans, vx, cnt, frames, clip_off, pitch_arr, pstarted ? pit.item + 1 : my_a, my_b);
        pstarted = true;
        psrc = pit.src;
        prows = pit.rows;
      }
      if (prows > 0) {
        mbar_expect_tx_if(&bars[g], (uint32_t)pit.nbytes, l0);
        tma_bulk_g2s_if(stage + (size_t)(g * kRGrp + q) * kRStageB, psrc, (uint32_t)pit.nbytes, &bars[g], l0);
        psrc += pit.pitch;
        --prows;
      }
    }
    mbar_arrive_if(&bars[g], l0);
  };
  for (uint32_t g = 0; g < kRNGrp; ++g) issue_group(g);
  // consumer: rc = staged rows consumed; row rc sits in slot rc % kRDepth, group barrier (rc / kRGrp) % kRNGrp,
  // phase (rc / kRDepth) & 1
  uint32_t rc = 0;
  auto consume_slot = [&]() {   // row rc has been read (its bytes are in registers): advance, refill its group
    const uint32_t used = rc++;
    if ((used & (kRGrp - 1)) == kRGrp - 1) {
      __syncwarp();
      issue_group((used / kRGrp) % kRNGrp);
    }
  };
  auto wait_row = [&]() {       // once per group: the group's rows have landed
    if ((rc & (kRGrp - 1)) == 0) mbar_wait(&bars[(rc / kRGrp) % kRNGrp], (rc / kRDepth) & 1);
  };

  const int p = kp.p, m = kp.m, tp = kp.tp, D = kp.D;
  const bool vlane = lane < kRLanes;
  // H lane = (channel hc, row pair hi): rows hi and hi + kRHP of the block
  const int hc = lane < 3 * kRHP ? lane / kRHP : 2, hi = lane < 3 * kRHP ? lane % kRHP : kRHP - 1;
  const bool hlane = lane < 3 * kRHP;
  const float hsc = hc == 0 ? kp.scale[0] : (hc == 1 ? kp.scale[1] : kp.scale[2]);
  const float hbi = hc == 0 ? kp.bias[0] : (hc == 1 ? kp.bias[1] : kp.bias[2]);
  const float hlo = hc == 0 ? kp.lo[0] : (hc == 1 ? kp.lo[1] : kp.lo[2]);
  const float hhi = hc == 0 ? kp.hi[0] : (hc == 1 ? kp.hi[1] : kp.hi[2]);
  const __nv_bfloat162 hlo2 = hc == 0 ? kp.lo2[0] : (hc == 1 ? kp.lo2[1] : kp.lo2[2]);
  const __nv_bfloat162 hhi2 = hc == 0 ? kp.hi2[0] : (hc == 1 ? kp.hi2[1] : kp.hi2[2]);
  const float2* hrow = reinterpret_cast<const float2*>(iP) + (size_t)(hc * kRHP + hi) * kRS;
  // staged output rows of this H lane (channel plane hc, block rows hi and hi + kRHP) and their bf16 swizzles
  const int orow0 = hc * kRHR + hi, orow1 = orow0 + kRHP;
  const int osw0 = kF32 ? 0 : 2 * ((orow0 >> 2) & 3), osw1 = kF32 ? 0 : 2 * ((orow1 >> 2) & 3);
  int cached_k = -1, cached_st = -1;
  int hstart = 0;

  for (int64_t item = my_a; item < my_b; ++item) {
    const RItem it = ring_item(plans, vx, cnt, item);
    const vp_clip_plan pl = plans[it.k];
    const int in_h = pl.in_h, out_h = pl.out_h, in_w = pl.in_w, out_w = pl.out_w;
    const int ws = ring_strip_width(in_w, out_w);
    const int j0 = it.st * ws, jn = min(ws, out_w - j0);
    const int pl0 = strip_pl(in_w, out_w, j0);
    const int pa = pl0 & ~15;
    const int soff = 3 * (pl0 - pa) + 12 * lane;       // this lane's bytes in a staged row
    void* pv = pl.is_image ? pv_img : pv_vid;
    const int64_t cap = pl.is_image ? img_cap : vid_cap;
    const bool writable = pv != nullptr && pl.patch_offset + (int64_t)pl.grid_t * pl.grid_h * pl.grid_w <= cap;

    // ---- horizontal table of (clip, strip): per footprint pixel q the weights of its live columns in slot
    //      order (column jj -> slot jj % 5) and the pixel's intermediate position; per column its window end ----
    if (it.k != cached_k || it.st != cached_st) {
      __syncwarp();
      for (int q = lane; q < kRS; q += kRT) {
        hw4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        hw2[q] = make_float2(0.f, __int_as_float(ipos(q < kRingPx ? q : 0)));
      }
      __syncwarp();
      for (int jj = lane; jj < jn; jj += kRT) {
        const Win w = window_of(in_w, out_w, j0 + jj);
        double s = 0.0;
        for (int x = w.x0; x < w.x1; ++x) s += keys_d(((double)x - w.c + 0.5) * w.inv);
        const double inv = s != 0.0 ? 1.0 / s : 1.0;
        hx1[jj] = min(w.x1 - pl0, kRingPx);
        const int slot = jj % kRing;
        for (int x = w.x0; x < w.x1; ++x) {
          const int q = x - pl0;
          if (q < 0 || q >= kRingPx) continue;
          const float wt = (float)(keys_d(((double)x - w.c + 0.5) * w.inv) * inv);
          if (slot < 4) reinterpret_cast<float*>(&hw4[q])[slot] = wt;
          else hw2[q].x = wt;
        }
      }
      if (lane == 0) hx1[jn] = 0x7fffffff;
      __syncwarp();
      hstart = window_of(in_w, out_w, j0).x0 - pl0;
      cached_k = it.k;
      cached_st = it.st;
    }
    const VTab T = vtab_at(vt, vt_owner[it.j]);

    // ---- output addressing (O8) ----
    const int f = it.f;
    const int last_slot = (f == pl.n_frames - 1) ? pl.grid_t * tp - 1 : f;   // O7: frame n-1 fills the pads
    const int nslots = last_slot - f + 1;
    const int g0 = f / tp, ti0 = f - g0 * tp;
    const int gh = pl.grid_h, gw = pl.grid_w;
    const int64_t group_stride = (int64_t)(gh / m) * (gw / m) * m * m * D;
    const int64_t tbase = (pl.patch_offset + (int64_t)g0 * (gh / m) * (gw / m) * m * m) * D + (int64_t)ti0 * p * p;
    const int64_t cstride = (int64_t)tp * p * p;

    // flush p-block jg >> 4 of the current H block: its rows x 3 channels x the strip's 16-B chunks
    // (every staged output element goes to each temporal slot it fills, O7)
    int nrows_cur = 0;
    auto flush = [&](int jg) {
      __syncwarp();
      const int pb = jg >> 4, clo = max(j0, jg & ~15) - 16 * pb, chi = jg + 1 - 16 * pb;
      const int64_t pboff = ((int64_t)(pb / m) * m * m + pb % m) * D;
      constexpr int kCh = kF32 ? 4 : 2, kCPx = 16 / kCh;   // 16-B chunks per 16-px row, px per chunk
      for (int u = lane; u < 3 * kRHR * kCh; u += kRT) {
        const int c = u / (kRHR * kCh), rem = u - c * (kRHR * kCh), rr = rem / kCh, q = rem - rr * kCh;
        if (!writable || rr >= nrows_cur || q * kCPx < clo || (q + 1) * kCPx > chi) continue;
        const int orow = c * kRHR + rr;
        const unsigned char* sp2 = ost + (size_t)orow * Cfg::OSTRIDE;
        const int sw = kF32 ? 0 : 2 * ((orow >> 2) & 3);      // bf16: 8-B granules (4q, 4q+2) ^ sw
        const float2 lo = *reinterpret_cast<const float2*>(sp2 + (kF32 ? 16 * q : 4 * ((4 * q) ^ sw)));
        const float2 hi2v = *reinterpret_cast<const float2*>(sp2 + (kF32 ? 16 * q + 8 : 4 * ((4 * q + 2) ^ sw)));
        const float4 v4 = make_float4(lo.x, lo.y, hi2v.x, hi2v.y);
        int64_t idx = rbase[rr] + pboff + c * cstride + q * kCPx;
        for (int s2 = 0, ti = ti0; s2 < nslots; ++s2) {
          if (kF32) *reinterpret_cast<float4*>(reinterpret_cast<float*>(pv) + idx) = v4;
          else *reinterpret_cast<float4*>(reinterpret_cast<__nv_bfloat16*>(pv) + idx) = v4;
          if (++ti == tp) { ti = 0; idx += group_stride - (int64_t)(tp - 1) * p * p; }
          else idx += (int64_t)p * p;
        }
      }
      __syncwarp();
    };

    VAcc acc[kRing];
#pragma unroll
    for (int s = 0; s < kRing; ++s) {
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[s].rg[q] = make_float2(0.f, 0.f);
      acc[s].b[0] = acc[s].b[1] = make_float2(0.f, 0.f);
    }
    int y = 0;
    for (int i0 = 0; i0 < out_h; i0 += kRHR) {
      const int nrows = min(kRHR, out_h - i0);
      nrows_cur = nrows;
      // ============================== V phase: output rows i0 .. i0+nrows-1.  Output row i lives in ring
      // slot i % 5; unrolling the output-row loop by 5 makes each retire's slot static.  For row i the
      // source rows up to its window end y1_i are consumed (each FMA'd into all 5 slots, weights in slot
      // order), then the row retires into the pair planes.
      for (int ib = i0; ib < i0 + nrows; ib += kRing) {
        int yends[kRing];
#pragma unroll
        for (int u = 0; u < kRing; ++u) yends[u] = __ldg(T.y1 + min(ib + u, out_h - 1));
#define VP_VROW(U)                                                                                  \
        if (ib + U < out_h) {                                                                       \
          for (; y < yends[U]; ++y) {                                                               \
            wait_row();                                                                             \
            const uint32_t* sp = reinterpret_cast<const uint32_t*>(stage + (rc % kRDepth) * kRStageB + soff); \
            const uint32_t r0 = sp[0], r1 = sp[1], r2 = sp[2];                                      \
            const float4 wa = __ldg(T.w4 + y);                                                      \
            const float wb = __ldg(T.w1 + y);                                                       \
            float2 crg[4], cb[2];                                                                   \
            cvt12(r0, r1, r2, crg, cb);        /* consumes the staged bytes before the refill */    \
            consume_slot();                                                                         \
            const float wv[kRing] = {wa.x, wa.y, wa.z, wa.w, wb};                                   \
            _Pragma("unroll") for (int s = 0; s < kRing; ++s) {                                     \
              const float2 ww = make_float2(wv[s], wv[s]);                                          \
              _Pragma("unroll") for (int q = 0; q < 4; ++q) acc[s].rg[q] = __ffma2_rn(ww, crg[q], acc[s].rg[q]); \
              acc[s].b[0] = __ffma2_rn(ww, cb[0], acc[s].b[0]);                                     \
              acc[s].b[1] = __ffma2_rn(ww, cb[1], acc[s].b[1]);                                     \
            }                                                                                       \
          }                                                                                         \
          {                                                                                         \
            const int rr = ib + U - i0;        /* pair rr % kRHP, half rr / kRHP */                 \
            float* dst = iP + ((size_t)(rr % kRHP) * kRS + lane) * 2 + rr / kRHP;                   \
            constexpr size_t kPl = (size_t)kRHP * kRS * 2;   /* channel plane stride (floats) */    \
            if (vlane) {                                                                            \
              _Pragma("unroll") for (int q = 0; q < 4; ++q) {                                       \
                dst[(size_t)q * kRLanes * 2] = acc[U].rg[q].x;                                      \
                dst[kPl + (size_t)q * kRLanes * 2] = acc[U].rg[q].y;                                \
              }                                                                                     \
              dst[2 * kPl] = acc[U].b[0].x;                                                         \
              dst[2 * kPl + (size_t)kRLanes * 2] = acc[U].b[0].y;                                   \
              dst[2 * kPl + (size_t)2 * kRLanes * 2] = acc[U].b[1].x;                               \
              dst[2 * kPl + (size_t)3 * kRLanes * 2] = acc[U].b[1].y;                               \
            }                                                                                       \
            _Pragma("unroll") for (int q = 0; q < 4; ++q) acc[U].rg[q] = make_float2(0.f, 0.f);     \
            acc[U].b[0] = acc[U].b[1] = make_float2(0.f, 0.f);                                      \
          }                                                                                         \
        }
        VP_VROW(0) VP_VROW(1) VP_VROW(2) VP_VROW(3) VP_VROW(4)
#undef VP_VROW
      }
      __syncwarp();

      // ============================== H phase: lane (hc, hi) walks the footprint pixels for rows hi, hi+kRHP.
      // Column jj lives in slot jj % 5; the column loop is unrolled by 10 (static slot and pair parity).
      {
        if (lane < kRHR) {   // destination row bases of the block's rows (O8, without the column part)
          const int i = i0 + min(lane, nrows - 1);
          const int hb = i / (m * p), mh = (i / p) % m, py = i % p;
          rbase[lane] = tbase + ((int64_t)hb * (gw / m) * m * m + (int64_t)mh * m) * D + (int64_t)py * p;
        }
        float2 ha[kRing];
#pragma unroll
        for (int s = 0; s < kRing; ++s) ha[s] = make_float2(0.f, 0.f);
        float2 pend = make_float2(0.f, 0.f);     // normalised even column (rows hi, hi + kRHP)
        int x = hstart;
        for (int jj0 = 0; jj0 < jn; jj0 += 2 * kRing) {
#define VP_HCOL(V)                                                                                  \
          if (jj0 + V < jn) {                                                                       \
            const int xend = hx1[jj0 + V];                                                          \
            for (; x < xend; ++x) {                                                                 \
              const float4 a4 = hw4[x];                                                             \
              const float2 a2 = hw2[x];                                                             \
              const float a1 = a2.x;                                                                \
              const float2 d = hrow[__float_as_int(a2.y)];                                          \
              ha[0] = __ffma2_rn(make_float2(a4.x, a4.x), d, ha[0]);                                \
              ha[1] = __ffma2_rn(make_float2(a4.y, a4.y), d, ha[1]);                                \
              ha[2] = __ffma2_rn(make_float2(a4.z, a4.z), d, ha[2]);                                \
              ha[3] = __ffma2_rn(make_float2(a4.w, a4.w), d, ha[3]);                                \
              ha[4] = __ffma2_rn(make_float2(a1, a1), d, ha[4]);                                    \
            }                                                                                       \
            {                                                                                       \
              constexpr int S = V % kRing;                                                          \
              const float2 nv = __ffma2_rn(ha[S], make_float2(hsc, hsc), make_float2(hbi, hbi)); /* O6 */ \
              ha[S] = make_float2(0.f, 0.f);                                                        \
              if ((V & 1) == 0) {                                                                   \
                pend = nv;                                                                          \
              } else {                                                                              \
                const int jg = j0 + jj0 + V;                  /* global column (odd) */             \
                const int pr = (jg & 15) >> 1;                /* column pair within the p-block */  \
                if (hlane) {                                                                        \
                  unsigned char* o0 = ost + (size_t)orow0 * Cfg::OSTRIDE;                          \
                  unsigned char* o1 = ost + (size_t)orow1 * Cfg::OSTRIDE;                          \
                  if (kF32) {                  /* C12 clamp in the output domain */                 \
                    *reinterpret_cast<float2*>(o0 + 8 * pr) =                                       \
                        make_float2(fminf(fmaxf(pend.x, hlo), hhi), fminf(fmaxf(nv.x, hlo), hhi));  \
                    *reinterpret_cast<float2*>(o1 + 8 * pr) =                                       \
                        make_float2(fminf(fmaxf(pend.y, hlo), hhi), fminf(fmaxf(nv.y, hlo), hhi));  \
                  } else {                                                                          \
                    *reinterpret_cast<__nv_bfloat162*>(o0 + 4 * (pr ^ osw0)) =                      \
                        __hmin2(__hmax2(__floats2bfloat162_rn(pend.x, nv.x), hlo2), hhi2);          \
                    *reinterpret_cast<__nv_bfloat162*>(o1 + 4 * (pr ^ osw1)) =                      \
                        __hmin2(__hmax2(__floats2bfloat162_rn(pend.y, nv.y), hlo2), hhi2);          \
                  }                                                                                 \
                }                                                                                   \
                if ((jg & 15) == 15 || jj0 + V == jn - 1) flush(jg);                                \
              }                                                                                     \
            }                                                                                       \
          }
          VP_HCOL(0) VP_HCOL(1) VP_HCOL(2) VP_HCOL(3) VP_HCOL(4)
          VP_HCOL(5) VP_HCOL(6) VP_HCOL(7) VP_HCOL(8) VP_HCOL(9)
#undef VP_HCOL
        }
      }
      __syncwarp();
    }
    // source rows below the last window keep the staging ring in step
    for (; y < in_h; ++y) {
      wait_row();
      __syncwarp();
      consume_slot();
    }
  }
}

// ---------------------------------------------------------------- per-clip vertical tables
// ring_owner_kernel (1 CTA): owner[j] = the last ring-list position <= j whose clip starts a run of equal
// vertical geometry (in_h, out_h) -- consecutive clips of equal geometry share one table.
constexpr int kOwnT = 1024;
__global__ void __launch_bounds__(kOwnT)
ring_owner_kernel(const vp_clip_plan* __restrict__ plans, const int* __restrict__ list, const int64_t* __restrict__ meta,
                  int* __restrict__ owner) {
  __shared__ int wmax[kOwnT / 32];
  __shared__ int carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cnt = (int)meta[0];
  if (tid == 0) carry = 0;
  __syncthreads();
  for (int c0 = 0; c0 < cnt; c0 += kOwnT) {
    const int j = c0 + tid;
    int v = 0;
    if (j < cnt) {
      const vp_clip_plan& a = plans[list[j]];
      bool fresh = j == 0;
      if (!fresh) {
        const vp_clip_plan& b = plans[list[j - 1]];
        fresh = a.in_h != b.in_h || a.out_h != b.out_h;
      }
      v = fresh ? j : 0;
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v = max(v, u);
    }
    if (lane == 31) wmax[warp] = v;
    __syncthreads();
    int pre = carry;
    for (int w = 0; w < warp; ++w) pre = max(pre, wmax[w]);
    v = max(v, pre);
    if (j < cnt) owner[j] = v;
    __syncthreads();
    if (tid == kOwnT - 1) carry = v;
    __syncthreads();
  }
}

// ring_vtables_kernel: for every owner position j, per source row y the weights of its live output rows in
// slot order (row i -> slot i % 5; 0 where not live) and per output row i its window end y1.
// Task = (list position j, chunk of kVtT rows); only owner positions compute.
constexpr int kVtT = 64;
constexpr int kVtChunks = (kRingInHMax + kVtT - 1) / kVtT;
__global__ void __launch_bounds__(kVtT)
ring_vtables_kernel(const vp_clip_plan* __restrict__ plans, const int* __restrict__ list,
                    const int64_t* __restrict__ meta, const int* __restrict__ owner, char* __restrict__ vt) {
  const int cnt = (int)meta[0];
  for (int64_t task = blockIdx.x; task < (int64_t)cnt * kVtChunks; task += gridDim.x) {
    const int j = (int)(task / kVtChunks), chunk = (int)(task % kVtChunks);
    if (owner[j] != j) continue;
    const vp_clip_plan& pl = plans[list[j]];
    const int in_h = pl.in_h, out_h = pl.out_h;
    if (chunk * kVtT >= in_h) continue;
    char* b = vt + (size_t)j * kVTabBytes;
    float4* w4 = reinterpret_cast<float4*>(b);
    float* w1 = reinterpret_cast<float*>(b + (size_t)16 * kRingInHMax);
    int* y1 = reinterpret_cast<int*>(b + (size_t)20 * kRingInHMax);
    const int yy = chunk * kVtT + threadIdx.x;
    if (yy < out_h) y1[yy] = window_of(in_h, out_h, yy).x1;
    const double sc = (double)in_h / (double)out_h;
    const double sup = 2.0 * (sc > 1.0 ? sc : 1.0);
    if (yy < in_h) {
      // first output row whose window has not ended before yy
      int i = (int)floor(((double)yy - sup - 0.5) / sc - 0.5);
      if (i < 0) i = 0;
      if (i > out_h) i = out_h;
      while (i > 0 && window_of(in_h, out_h, i - 1).x1 > yy) --i;
      while (i < out_h && window_of(in_h, out_h, i).x1 <= yy) ++i;
      float wv[kRing] = {0.f, 0.f, 0.f, 0.f, 0.f};
      for (int r = 0; r < kRing && i + r < out_h; ++r) {
        const Win w = window_of(in_h, out_h, i + r);
        if (w.x0 > yy || yy >= w.x1) continue;
        double s = 0.0;
        for (int x = w.x0; x < w.x1; ++x) s += keys_d(((double)x - w.c + 0.5) * w.inv);
        wv[(i + r) % kRing] = (float)(keys_d(((double)yy - w.c + 0.5) * w.inv) / (s != 0.0 ? s : 1.0));
      }
      w4[yy] = make_float4(wv[0], wv[1], wv[2], wv[3]);
      w1[yy] = wv[4];
    }
  }
}

bool g_rattr[2] = {};

template <bool kF32>
void launch_ring_t(const FKParams& kp, const vp_clip_plan* plans, const VIdx& vx, const uint8_t* frames,
                   const int64_t* coff, const int64_t* pitch, void* pi, int64_t icap, void* pvv, int64_t vcap,
                   const char* vt, const int* owner, int num_sms, cudaStream_t s) {
  using Cfg = RingCfg<kF32>;
  auto kern = resize_ring_kernel<kF32>;
  if (!g_rattr[kF32]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM);
    g_rattr[kF32] = true;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRT, Cfg::SMEM);
  if (per_sm < 1) per_sm = 1;
  kern<<<num_sms * per_sm, kRT, Cfg::SMEM, s>>>(kp, plans, vx, frames, coff, pitch, pi, icap, pvv, vcap, vt, owner);
}

}  // namespace

size_t ring_vtable_bytes() { return kVTabBytes; }

cudaError_t launch_resize_ring(const FKParams& kp, const vp_clip_plan* plans, const VIdx& vx, const uint8_t* frames,
                               const int64_t* coff, const int64_t* pitch, void* pi, int64_t icap, void* pvv,
                               int64_t vcap, int n, void* vt, int* vt_owner, int num_sms, cudaStream_t s) {
  (void)n;
  ring_owner_kernel<<<1, kOwnT, 0, s>>>(plans, vx.list, vx.meta, vt_owner);
  ring_vtables_kernel<<<num_sms * 8, kVtT, 0, s>>>(plans, vx.list, vx.meta, vt_owner, reinterpret_cast<char*>(vt));
  if (kp.out_f32) launch_ring_t<true>(kp, plans, vx, frames, coff, pitch, pi, icap, pvv, vcap, (const char*)vt, vt_owner,
                                      num_sms, s);
  else launch_ring_t<false>(kp, plans, vx, frames, coff, pitch, pi, icap, pvv, vcap, (const char*)vt, vt_owner,
                            num_sms, s);
  return cudaGetLastError();
}

}  // namespace vp
