// vp_k3_common.cuh -- device helpers shared by the K3 kernels (vp_resize_fast.cu, vp_resize_team.cu, vp_resize.cu):
// normalisation parameters, mbarrier / TMA-bulk PTX wrappers, the AA-bicubic window (C10) and the
// per-variant work index.  Private to the CUDA path; nothing here is shared with oracle/.
#pragma once
#include "vp_internal.cuh"
#include <cuda_bf16.h>

namespace vp {

struct FKParams {
  int p, m, tp, D;
  float scale[3], bias[3];
  float lo[3], hi[3];               // output-domain clamp bounds: bias, fma(255, scale, bias)
  __nv_bfloat162 lo2[3], hi2[3];    // the same, RNE to bf16, duplicated
  int out_f32;                      // VP_OUT_F32
};

// ---------------------------------------------------------------- PTX helpers (mbarrier / TMA bulk)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// Shared-memory accesses at explicit 32-bit shared addresses (volatile: ordered with the mbarrier waits / barriers
// that guard the data; the address arithmetic folds into [R + imm] with no generic-to-shared conversion).
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_f4(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
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
// Warp-uniform wait (every lane tests the same barrier phase in one instruction, so the retry branch is uniform:
// bra.uni spares ptxas the divergence bookkeeping around the loop).  kHint > 0 adds a suspend-time hint (ns).
template <int kHint = 0>
__device__ __forceinline__ void mbar_wait_uni(uint64_t* bar, uint32_t parity) {
  if (kHint > 0)
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAITH_%=:\n"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@!P1 bra.uni WAITH_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "n"(kHint)
        : "memory");
  else
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAITU_%=:\n"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra.uni WAITU_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// Wait with a suspend-time hint: the thread may be suspended (not re-issuing try_wait) until the phase
// completes or the hint expires -- for consumers that routinely wait long (H warps waiting on V rows), so that
// spinning does not take issue slots from the warps doing the work.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAITS_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@!P1 bra WAITS_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(1000000)
      : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Predicated forms (the predicate is a per-lane value; the instruction stream stays warp-uniform, so a
// warp-uniform producer issues from one lane without a divergent branch).
__device__ __forceinline__ void mbar_expect_tx_if(uint64_t* bar, uint32_t bytes, bool pred) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %2, 0;\n"
      "@p mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n}" ::"r"(smem_u32(bar)),
      "r"(bytes), "r"((int)pred)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_if(uint64_t* bar, bool pred) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %1, 0;\n"
      "@p mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n}" ::"r"(smem_u32(bar)),
      "r"((int)pred)
      : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s_if(void* dst, const void* src, uint32_t bytes, uint64_t* bar, bool pred) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "@p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n}" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "r"((int)pred)
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

// Window of output index i on an in->out axis (C10), trimmed of exact-zero end taps (zero taps add
// exactly 0 to the sum; trimming makes identity axes 1-tap).  x0, x1 (exclusive), centre c, 1/fs.
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
  while (w.x1 - w.x0 > 1 && keys_d(((double)w.x0 - w.c + 0.5) * w.inv) == 0.0) ++w.x0;
  while (w.x1 - w.x0 > 1 && keys_d(((double)(w.x1 - 1) - w.c + 0.5) * w.inv) == 0.0) --w.x1;
  return w;
}

// Per-variant work index (built per call by variant_index_kernel): the variant's clips in batch order
// (list), the exclusive prefix of their item counts (off, count+1 entries) and meta = {count, items}.
// Every CTA of a variant's launch takes a contiguous slice of that variant's items only.
struct VIdx {
  const int* list;
  const int64_t* off;
  const int64_t* meta;
};
__device__ __forceinline__ int vfind(const VIdx& vx, int cnt, int64_t item) {   // last j with off[j] <= item
  int lo = 0, hi = cnt - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (vx.off[mid] <= item) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Per-variant work-index slots (variant_index_kernel): MILD, MEDIUM, STRONG, COPY, TEAM, WIDE, TEAML, U8.
constexpr int kNSlots = 8;

// Caller workspace of vp_resize_normalize_patchify (resize_ws_layout): the per-variant work index and the
// KV_TEAM per-clip tables.  Nothing persists between calls.
struct ResizeWs {
  size_t bytes;
  int* list;          // [kNSlots][n]
  int64_t* off;       // [kNSlots][n+1]
  int64_t* meta;      // [kNSlots][4]: clips, items, row bands per frame (team slots), unused
  int* alias;         // [n]  clip -> first clip of its run of equal (in_h, out_h) TEAM / WIDE clips (table owner)
  int* tflag;         // [n]  table flags (a non-negligible 5th live row)
  float4* vtab;       // [n][kTabInH]
  int* y1tab;         // [n][kTabOutStride]
  int2* u8prec;       // [n]  KV_U8 coefficient precision (horizontal, vertical)
};
ResizeWs resize_ws_layout(int n, void* base);
VIdx ws_vidx(const ResizeWs& w, int n, int slot);
int device_sms(int dev);
cudaError_t launch_index(const vp_clip_plan* plans, int n, const int64_t* coff, const int64_t* pitch,
                         const ResizeWs& w, int num_sms, cudaStream_t s);
cudaError_t launch_team(const FKParams& kp, const vp_clip_plan* plans, int n, const ResizeWs& w, const uint8_t* frames,
                        const int64_t* coff, const int64_t* pitch, void* pi, int64_t icap, void* pvv, int64_t vcap,
                        int32_t* clip_status, int dev, int num_sms, unsigned mask, cudaStream_t s);
cudaError_t launch_fast_variants(const FKParams& kp, const vp_clip_plan* plans, int n, const ResizeWs& w,
                                 const uint8_t* frames, const int64_t* coff, const int64_t* pitch, void* pi,
                                 int64_t icap, void* pvv, int64_t vcap, int dev, int num_sms, unsigned mask,
                                 cudaStream_t s);
FKParams make_fkparams(const vp_params* p);
cudaError_t launch_u8(const FKParams& kp, const vp_clip_plan* plans, int n, const ResizeWs& w, const uint8_t* frames,
                      const int64_t* coff, const int64_t* pitch, void* pi, int64_t icap, void* pvv, int64_t vcap,
                      int num_sms, cudaStream_t s);

}  // namespace vp
