// vp_resize_fast.cu -- K3 fast path: streaming fused AA-bicubic resize + clamp + normalise +
// temporal pad + patchify (O4-O9) for the common ratios (KV_MILD / KV_STRONG, see vp_internal.cuh).
//
// Work item = (clip, source frame f, strip of Ws output columns); a CTA walks the item's source
// rows top to bottom once:
//   * producer warp: streams each source row's footprint bytes (16-B aligned, <= 512 / 1024 B) into a
//     16-slot shared-memory ring with cp.async.bulk (TMA bulk copy) + mbarrier complete_tx, running
//     ahead across items;
//   * NCW consumer warps, vertical pass: lane L owns 4 consecutive footprint bytes; every source row is
//     read from smem once (LDS.32), converted once (I2F.U8) and FMA'd (FFMA2) into the <= 8 live output
//     rows held in a register ring acc[8] -- uniform per-row control (meta[y]: first live row, live
//     count, retiring count) dispatched with one jump-table switch per row, so no dynamic register
//     indexing and no wasted FMAs;
//   * retired output rows (fp32, footprint-wide) go to a small smem buffer; every 4 rows the consumers
//     run the horizontal pass (weights in registers for MILD), clamp, normalise (one FFMA), round to
//     bf16/f32 and store straight into the HF patch layout -- every output element written once, to
//     every temporal slot the frame fills (odd-n padding, images).
// Tables (per clip, cached across a CTA's consecutive items): vertical windows as a compact
// per-source-row list (meta + weights), weights computed in f64 and stored fp32.
#include "vp_internal.cuh"
#include <cuda_bf16.h>

namespace vp {
namespace {

constexpr int kSlots = 16;        // source-row ring depth (TMA in flight)
constexpr int kCapR = 8;          // retired-row buffer (rows)
constexpr int kQH = 4;            // horizontal pass every 4 retired rows

struct FKParams {
  int p, m, tp, D;
  float scale[3], bias[3];
};

// ---------------------------------------------------------------- PTX helpers (mbarrier / TMA bulk)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ double keys_d(double x) {
  const double a = -0.5;
  x = fabs(x);
  if (x < 1.0) return ((a + 2.0) * x - (a + 3.0)) * x * x + 1.0;
  if (x < 2.0) return (((x - 5.0) * x + 8.0) * x - 4.0) * a;
  return 0.0;
}

// Window of output index i on an in->out axis (C10): x0, x1 (exclusive), centre c, 1/fs.
struct Win {
  int x0, x1;
  double c, inv;
};
__device__ __forceinline__ Win window_of(int in, int out, int i) {
  const double scale = (double)in / (double)out;
  const double fs = scale > 1.0 ? scale : 1.0;
  const double support = 2.0 * fs;
  Win w;
  w.inv = 1.0 / fs;
  w.c = ((double)i + 0.5) * scale;
  w.x0 = (int)(w.c - support + 0.5);
  if (w.x0 < 0) w.x0 = 0;
  w.x1 = (int)(w.c + support + 0.5);
  if (w.x1 > in) w.x1 = in;
  return w;
}

__device__ __forceinline__ int find_clip_f(const vp_clip_plan* __restrict__ plans, int n, int64_t item) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (plans[mid].tile_offset <= item) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Item decode shared by producer and consumers.
struct Item {
  int k;            // clip
  int f;            // source frame
  int strip, ws, j0, jn;   // strip index, strip width, first column, columns in this strip
  int64_t clip_end; // first item after this clip
  bool mine;
};

__device__ __forceinline__ bool clip_is_mine(const vp_clip_plan& pl, int variant, int64_t coff, int64_t pitch) {
  return pl.status == VP_OK && pl.kernel_variant == variant && ((coff | pitch) & 15) == 0 && pl.tile_count > 0;
}

// ---------------------------------------------------------------- the vertical ring (switch dispatch)
// acc[r] = {bytes 0,1} and acc[r+8] = {bytes 2,3} of output row in slot r (slot = row & 7)
#define VP_FMA2(A, W, F)                                                       \
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(A) : "l"(F), "l"(W))

__device__ __forceinline__ unsigned long long pack2(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 unpack2(unsigned long long v) {
  float2 r;
  asm("mov.b64 {%0,%1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}

template <int BASE, int CNT>
__device__ __forceinline__ void ring_contrib(unsigned long long (&acc)[16], const float* __restrict__ w,
                                             unsigned long long f01, unsigned long long f23) {
#pragma unroll
  for (int r = 0; r < CNT; ++r) {
    constexpr int dummy = 0;
    (void)dummy;
    const int slot = (BASE + r) & 7;
    const float wr = w[r];
    const unsigned long long ww = pack2(wr, wr);
    VP_FMA2(acc[slot], ww, f01);
    VP_FMA2(acc[slot + 8], ww, f23);
  }
}

#define VP_RC(B)                                                              \
  case B * 16 + 0: break;                                                     \
  case B * 16 + 1: ring_contrib<B, 1>(acc, w, f01, f23); break;               \
  case B * 16 + 2: ring_contrib<B, 2>(acc, w, f01, f23); break;               \
  case B * 16 + 3: ring_contrib<B, 3>(acc, w, f01, f23); break;               \
  case B * 16 + 4: ring_contrib<B, 4>(acc, w, f01, f23); break;               \
  case B * 16 + 5: ring_contrib<B, 5>(acc, w, f01, f23); break;               \
  case B * 16 + 6: ring_contrib<B, 6>(acc, w, f01, f23); break;               \
  case B * 16 + 7: ring_contrib<B, 7>(acc, w, f01, f23); break;               \
  case B * 16 + 8: ring_contrib<B, 8>(acc, w, f01, f23); break;

__device__ __forceinline__ void ring_step(unsigned long long (&acc)[16], int code, const float* __restrict__ w,
                                          unsigned long long f01, unsigned long long f23) {
  switch (code) {
    VP_RC(0) VP_RC(1) VP_RC(2) VP_RC(3) VP_RC(4) VP_RC(5) VP_RC(6) VP_RC(7)
    default: break;
  }
}

template <int BASE, int NRET>
__device__ __forceinline__ void ring_retire(unsigned long long (&acc)[16], float* __restrict__ vbuf, int row0,
                                            int fpf, int lane_f, bool active) {
#pragma unroll
  for (int r = 0; r < NRET; ++r) {
    const int slot = (BASE + r) & 7;
    if (active) {
      float2 a = unpack2(acc[slot]), b = unpack2(acc[slot + 8]);
      float4* dst = reinterpret_cast<float4*>(vbuf + ((row0 + r) & (kCapR - 1)) * fpf + lane_f);
      *dst = make_float4(a.x, a.y, b.x, b.y);
    }
    acc[slot] = 0ull;
    acc[slot + 8] = 0ull;
  }
}

#define VP_RR(B)                                                                  \
  case B * 4 + 1: ring_retire<B, 1>(acc, vbuf, row0, fpf, lane_f, active); break; \
  case B * 4 + 2: ring_retire<B, 2>(acc, vbuf, row0, fpf, lane_f, active); break; \
  case B * 4 + 3: ring_retire<B, 3>(acc, vbuf, row0, fpf, lane_f, active); break;

__device__ __forceinline__ void ring_retire_dispatch(unsigned long long (&acc)[16], int code, float* __restrict__ vbuf,
                                                     int row0, int fpf, int lane_f, bool active) {
  switch (code) {
    VP_RR(0) VP_RR(1) VP_RR(2) VP_RR(3) VP_RR(4) VP_RR(5) VP_RR(6) VP_RR(7)
    default: break;
  }
}

// ---------------------------------------------------------------- kernel
template <int VARIANT, bool kF32>
struct FastCfg {
  static constexpr int NCW = VARIANT == KV_MILD ? 4 : 8;           // consumer warps
  static constexpr int NC = NCW * 32;                               // consumer threads
  static constexpr int FPB = VARIANT == KV_MILD ? 512 : 1024;       // footprint bytes per row
  static constexpr int LHM = VARIANT == KV_MILD ? 12 : 40;          // horizontal taps bound
  static constexpr bool HREG = VARIANT == KV_MILD;                  // horizontal weights in registers
  static constexpr int UPT = VARIANT == KV_MILD ? 2 : 1;            // max (col,channel) units per thread
  static constexpr int MAXWS = (UPT * NC) / 3;                      // strip width bound from units
  static constexpr int VPAD = 3 * LHM + 16;                         // slack after each V row (floats)
  static constexpr int FPF = FPB + VPAD;                            // floats per retired row
  // smem layout (bytes)
  static constexpr size_t OFF_RING = 0;                                                   // kSlots*FPB u8
  static constexpr size_t OFF_VBUF = OFF_RING + (size_t)kSlots * FPB;                     // kCapR*FPF f32
  static constexpr size_t OFF_META = OFF_VBUF + (size_t)kCapR * FPF * 4;                  // kInHMax int2
  static constexpr size_t OFF_WL = OFF_META + (size_t)kInHMax * 8;                        // kWListMax f32
  static constexpr size_t OFF_WH = OFF_WL + (size_t)kWListMax * 4;                        // MAXWS*LHM f32
  static constexpr size_t OFF_HX = OFF_WH + (size_t)MAXWS * LHM * 4;                      // MAXWS int
  static constexpr size_t OFF_BAR = (OFF_HX + (size_t)MAXWS * 4 + 15) & ~(size_t)15;     // 2*kSlots u64
  static constexpr size_t OFF_MISC = OFF_BAR + 2 * kSlots * 8;
  static constexpr size_t SMEM = OFF_MISC + 64;
};

template <int VARIANT, bool kF32>
__global__ void __launch_bounds__(FastCfg<VARIANT, kF32>::NC + 32)
resize_fast_kernel(FKParams kp, const vp_clip_plan* __restrict__ plans, int n, const uint8_t* __restrict__ frames,
                   const int64_t* __restrict__ clip_off, const int64_t* __restrict__ pitch_arr, void* pv_img,
                   int64_t img_cap, void* pv_vid, int64_t vid_cap) {
  using Cfg = FastCfg<VARIANT, kF32>;
  extern __shared__ __align__(128) unsigned char smem[];
  uint8_t* ring = smem + Cfg::OFF_RING;
  float* vbuf = reinterpret_cast<float*>(smem + Cfg::OFF_VBUF);
  int2* meta = reinterpret_cast<int2*>(smem + Cfg::OFF_META);
  float* wl = reinterpret_cast<float*>(smem + Cfg::OFF_WL);
  float* wh = reinterpret_cast<float*>(smem + Cfg::OFF_WH);
  int* hx = reinterpret_cast<int*>(smem + Cfg::OFF_HX);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint64_t* empty = full + kSlots;
  int* misc = reinterpret_cast<int*>(smem + Cfg::OFF_MISC);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const bool producer = warp == Cfg::NCW;

  // item range of this CTA (contiguous slice of the batch's fast-item space)
  const int64_t it_begin = plans[0].tile_offset;
  const int64_t it_end = plans[n - 1].tile_offset + plans[n - 1].tile_count;
  const int64_t total = it_end - it_begin;
  const int64_t my_a = it_begin + total * blockIdx.x / gridDim.x;
  const int64_t my_b = it_begin + total * (blockIdx.x + 1) / gridDim.x;

  if (tid == 0) {
    for (int s = 0; s < kSlots; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cfg::NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < kCapR * Cfg::FPF; i += blockDim.x) vbuf[i] = 0.f;
  __syncthreads();

  if (producer) {
    // ------------------------------------------------------------ producer: TMA bulk row streaming
    if ((tid & 31) != 0) return;
    uint32_t slot = 0, phase = 0;
    int64_t item = my_a;
    while (item < my_b) {
      const int k = find_clip_f(plans, n, item);
      const vp_clip_plan pl = plans[k];
      const int64_t cend = pl.tile_offset + pl.tile_count;
      const int64_t coff = clip_off[k], pitch = pitch_arr[k];
      if (!clip_is_mine(pl, VARIANT, coff, pitch)) {
        item = cend;
        continue;
      }
      const int ws = fast_strip_width(pl.in_w, pl.out_w, VARIANT);
      const int nstrips = (pl.out_w + ws - 1) / ws;
      for (; item < cend && item < my_b; ++item) {
        const int64_t local = item - pl.tile_offset;
        const int f = (int)(local / nstrips), strip = (int)(local % nstrips);
        const int j0 = strip * ws, jn = min(ws, pl.out_w - j0);
        const Win wa = window_of(pl.in_w, pl.out_w, j0);
        const Win wb = window_of(pl.in_w, pl.out_w, j0 + jn - 1);
        const int b0 = (3 * wa.x0) & ~15;
        int b1 = (3 * wb.x1 + 15) & ~15;
        const int nbytes = b1 - b0;
        const uint8_t* src = frames + coff + (int64_t)f * pl.in_h * pitch + b0;
        for (int y = 0; y < pl.in_h; ++y) {
          mbar_wait(&empty[slot], phase ^ 1);
          mbar_arrive_expect_tx(&full[slot], (uint32_t)nbytes);
          tma_bulk_g2s(ring + (size_t)slot * Cfg::FPB, src + (int64_t)y * pitch, (uint32_t)nbytes, &full[slot]);
          if (++slot == kSlots) { slot = 0; phase ^= 1; }
        }
      }
    }
    return;
  }

  // ------------------------------------------------------------ consumers
  const int NC = Cfg::NC;
  const int p = kp.p, m = kp.m, tp = kp.tp, B = m * p;
  uint32_t slot = 0, phase = 0;
  int cached_clip = -1, cached_strip = -1;
  float hw[Cfg::HREG ? Cfg::UPT * Cfg::LHM : 1];
  int h_x[Cfg::UPT], h_c[Cfg::UPT], h_j[Cfg::UPT];
  int64_t item = my_a;
  while (item < my_b) {
    const int k = find_clip_f(plans, n, item);
    const vp_clip_plan pl = plans[k];
    const int64_t cend = pl.tile_offset + pl.tile_count;
    const int64_t coff = clip_off[k], pitch = pitch_arr[k];
    if (!clip_is_mine(pl, VARIANT, coff, pitch)) {
      item = cend;
      continue;
    }
    void* pv = pl.is_image ? pv_img : pv_vid;
    const int64_t cap = pl.is_image ? img_cap : vid_cap;
    const bool writable = pv != nullptr && pl.patch_offset + (int64_t)pl.grid_t * pl.grid_h * pl.grid_w <= cap;
    const int ws = fast_strip_width(pl.in_w, pl.out_w, VARIANT);
    const int nstrips = (pl.out_w + ws - 1) / ws;
    const int in_h = pl.in_h, out_h = pl.out_h;

    if (k != cached_clip) {
      // ---- vertical tables for this clip (K2), consumers only ----
      named_sync(1, NC);
      // A: 1/sum of each output row's weights (f32), aliased in vbuf
      float* invs = vbuf;
      for (int i = tid; i < out_h; i += NC) {
        const Win w = window_of(in_h, out_h, i);
        double s = 0.0;
        for (int y = w.x0; y < w.x1; ++y) s += keys_d(((double)y - w.c + 0.5) * w.inv);
        invs[i] = (float)(s != 0.0 ? 1.0 / s : 1.0);
      }
      // B: per source row: first live output row ia, live count, retiring count
      const double sc = (double)in_h / (double)out_h;
      const double sup = 2.0 * (sc > 1.0 ? sc : 1.0);
      for (int y = tid; y < in_h; y += NC) {
        // first i with x1_i > y: x1_i = int((i+0.5)s + sup + 0.5); estimate then correct
        int i = (int)floor(((double)y - sup - 0.5) / sc - 0.5);
        if (i < 0) i = 0;
        while (i > 0 && window_of(in_h, out_h, i - 1).x1 > y) --i;
        while (i < out_h && window_of(in_h, out_h, i).x1 <= y) ++i;
        int cnt = 0, nret = 0;
        for (int r = 0; r < kRing && i + r < out_h; ++r) {
          const Win w = window_of(in_h, out_h, i + r);
          if (w.x0 > y) break;
          ++cnt;
          if (w.x1 - 1 == y) ++nret;
        }
        meta[y] = make_int2(cnt, (i << 8) | (cnt << 4) | nret);
      }
      named_sync(1, NC);
      // C: exclusive scan of cnt over rows (single warp, serial over chunks of 32)
      if (warp == 0) {
        int carry = 0;
        for (int y0 = 0; y0 < in_h; y0 += 32) {
          const int y = y0 + (tid & 31);
          int v = y < in_h ? meta[y].x : 0, x = v;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(0xffffffffu, x, o);
            if ((tid & 31) >= o) x += t;
          }
          if (y < in_h) meta[y].x = carry + x - v;
          carry += __shfl_sync(0xffffffffu, x, 31);
        }
      }
      named_sync(1, NC);
      // D: weights
      for (int y = tid; y < in_h; y += NC) {
        const int2 me = meta[y];
        const int i0 = me.y >> 8, cnt = (me.y >> 4) & 15;
        for (int r = 0; r < cnt; ++r) {
          const Win w = window_of(in_h, out_h, i0 + r);
          wl[me.x + r] = (float)keys_d(((double)y - w.c + 0.5) * w.inv) * invs[i0 + r];
        }
      }
      named_sync(1, NC);
      for (int i = tid; i < kCapR * Cfg::FPF; i += NC) vbuf[i] = 0.f;
      cached_clip = k;
      cached_strip = -1;
    }

    for (; item < cend && item < my_b; ++item) {
      const int64_t local = item - pl.tile_offset;
      const int f = (int)(local / nstrips), strip = (int)(local % nstrips);
      const int j0 = strip * ws, jn = min(ws, pl.out_w - j0);
      const Win wa = window_of(pl.in_w, pl.out_w, j0);
      const Win wb = window_of(pl.in_w, pl.out_w, j0 + jn - 1);
      const int b0 = (3 * wa.x0) & ~15;
      const int nbytes = ((3 * wb.x1 + 15) & ~15) - b0;
      if (strip != cached_strip) {
        // ---- horizontal weights of this strip ----
        named_sync(1, NC);
        for (int jj = tid; jj < jn; jj += NC) {
          const Win w = window_of(pl.in_w, pl.out_w, j0 + jj);
          double s = 0.0, ww[Cfg::LHM];
#pragma unroll 1
          for (int l = 0; l < Cfg::LHM; ++l) {
            ww[l] = (w.x0 + l < w.x1) ? keys_d(((double)(w.x0 + l) - w.c + 0.5) * w.inv) : 0.0;
            s += ww[l];
          }
          const double r = s != 0.0 ? 1.0 / s : 1.0;
#pragma unroll 1
          for (int l = 0; l < Cfg::LHM; ++l) wh[jj * Cfg::LHM + l] = (float)(ww[l] * r);
          hx[jj] = 3 * w.x0 - b0;                  // float index of (x0, channel 0) in a V row
        }
        named_sync(1, NC);
        for (int u = 0; u < Cfg::UPT; ++u) {
          const int unit = tid + u * NC;           // unit = c * jn + jj (consecutive threads -> consecutive px)
          const int c = unit / jn, jj = unit - c * jn;
          h_c[u] = c < 3 ? c : -1;
          h_j[u] = jj;
          h_x[u] = c < 3 ? hx[jj] + c : 0;
          if (Cfg::HREG) {
#pragma unroll
            for (int l = 0; l < Cfg::LHM; ++l) hw[u * Cfg::LHM + l] = c < 3 ? wh[jj * Cfg::LHM + l] : 0.f;
          }
        }
        cached_strip = strip;
      }
      // slots filled by frame f (O7): f itself, and tp*gt-1 .. n for the last frame
      const int n_fr = pl.n_frames;
      const int last_slot = (f == n_fr - 1) ? pl.grid_t * tp - 1 : f;
      const int gh = pl.grid_h, gw = pl.grid_w;

      unsigned long long acc[16];
#pragma unroll
      for (int r = 0; r < 16; ++r) acc[r] = 0ull;
      const int lane_f = tid * 4;                   // this lane's float index within a V row
      const bool vactive = lane_f < nbytes;
      int retired = 0, done = 0;

      auto hpass = [&](int rows_to) {
        // rows [done, rows_to) are in vbuf (row i at slot i & (kCapR-1))
        named_sync(1, NC);
        if (writable) {
          for (int i = done; i < rows_to; ++i) {
            const float* vrow = vbuf + (i & (kCapR - 1)) * Cfg::FPF;
            const int hb = i / B, il = i - hb * B, mh = il / p, py = il - mh * p;
#pragma unroll
            for (int u = 0; u < Cfg::UPT; ++u) {
              const int c = h_c[u];
              if (c < 0) continue;
              const float* vp_ = vrow + h_x[u];
              float a = 0.f;
              if (Cfg::HREG) {
#pragma unroll
                for (int l = 0; l < Cfg::LHM; ++l) a = fmaf(hw[u * Cfg::LHM + l], vp_[3 * l], a);
              } else {
                const float* wr = wh + h_j[u] * Cfg::LHM;
#pragma unroll 8
                for (int l = 0; l < Cfg::LHM; ++l) a = fmaf(wr[l], vp_[3 * l], a);
              }
              a = fminf(fmaxf(a, 0.f), 255.f);                            // C12
              const float x = fmaf(a, kp.scale[c], kp.bias[c]);            // O6
              const int j = j0 + h_j[u];
              const int wbk = j / B, jl = j - wbk * B, mw = jl / p, px = jl - mw * p;
              for (int sl = f; sl <= last_slot; ++sl) {
                const int g = sl / tp, ti = sl - g * tp;
                const int64_t row = pl.patch_offset + (((int64_t)g * (gh / m) + hb) * (gw / m) + wbk) * m * m +
                                    mh * m + mw;
                const int64_t q = ((int64_t)(c * tp + ti) * p + py) * p + px;
                if (kF32) reinterpret_cast<float*>(pv)[row * kp.D + q] = x;
                else reinterpret_cast<__nv_bfloat16*>(pv)[row * kp.D + q] = __float2bfloat16_rn(x);
              }
            }
          }
        }
        done = rows_to;
        named_sync(1, NC);
      };

      for (int y = 0; y < in_h; ++y) {
        mbar_wait(&full[slot], phase);
        unsigned long long f01 = 0ull, f23 = 0ull;
        if (vactive) {
          const uint32_t raw = *reinterpret_cast<const uint32_t*>(ring + (size_t)slot * Cfg::FPB + lane_f);
          f01 = pack2((float)(raw & 0xffu), (float)((raw >> 8) & 0xffu));
          f23 = pack2((float)((raw >> 16) & 0xffu), (float)(raw >> 24));
        }
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(&empty[slot]);
        if (++slot == kSlots) { slot = 0; phase ^= 1; }
        const int2 me = meta[y];
        const int ia = me.y >> 8, cnt = (me.y >> 4) & 15, nret = me.y & 15;
        ring_step(acc, ((ia & 7) << 4) | cnt, wl + me.x, f01, f23);
        if (nret) {
          ring_retire_dispatch(acc, ((ia & 7) << 2) | nret, vbuf, ia, Cfg::FPF, lane_f, vactive);
          retired = ia + nret;
          if (retired - done >= kQH) hpass(retired);
        }
      }
      if (retired > done) hpass(retired);
    }
  }
  (void)misc;
}

int g_num_sms = 0;
bool g_attr[2][2] = {{false, false}, {false, false}};

template <int VARIANT, bool kF32>
void launch_fast(const FKParams& kp, const vp_clip_plan* plans, int n, const uint8_t* frames, const int64_t* coff,
                 const int64_t* pitch, void* pi, int64_t icap, void* pvv, int64_t vcap, cudaStream_t s) {
  using Cfg = FastCfg<VARIANT, kF32>;
  auto kern = resize_fast_kernel<VARIANT, kF32>;
  if (!g_attr[VARIANT][kF32]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM);
    g_attr[VARIANT][kF32] = true;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, Cfg::NC + 32, Cfg::SMEM);
  if (per_sm < 1) per_sm = 1;
  const int grid = g_num_sms * per_sm;
  kern<<<grid, Cfg::NC + 32, Cfg::SMEM, s>>>(kp, plans, n, frames, coff, pitch, pi, icap, pvv, vcap);
}

}  // namespace

// Launch both fast variants (each skips clips that are not its own).
void launch_resize_fast(const vp_params* p, const vp_clip_plan* plans, int n, const uint8_t* frames,
                        const int64_t* coff, const int64_t* pitch, void* pi, int64_t icap, void* pvv, int64_t vcap,
                        cudaStream_t s) {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  FKParams kp{};
  kp.p = p->patch_size;
  kp.m = p->merge_size;
  kp.tp = p->temporal_patch_size;
  kp.D = 3 * kp.tp * kp.p * kp.p;
  for (int c = 0; c < 3; ++c) {
    kp.scale[c] = (float)(1.0 / (255.0 * p->std[c]));
    kp.bias[c] = (float)(-p->mean[c] / p->std[c]);
  }
  if (p->out_dtype == VP_OUT_F32) {
    launch_fast<KV_MILD, true>(kp, plans, n, frames, coff, pitch, pi, icap, pvv, vcap, s);
    launch_fast<KV_STRONG, true>(kp, plans, n, frames, coff, pitch, pi, icap, pvv, vcap, s);
  } else {
    launch_fast<KV_MILD, false>(kp, plans, n, frames, coff, pitch, pi, icap, pvv, vcap, s);
    launch_fast<KV_STRONG, false>(kp, plans, n, frames, coff, pitch, pi, icap, pvv, vcap, s);
  }
}

}  // namespace vp
