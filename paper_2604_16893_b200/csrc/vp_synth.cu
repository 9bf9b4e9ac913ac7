// vp_synth.cu -- K5: synthetic u8 frame generator for tests and the bench (not the hot path,
// never inside a timed region).  Formulas identical to vp_inputs.frames_u8 (host), which the
// GPU tests check bit-exactly.
#include "vp_internal.cuh"

namespace vp {
namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// One thread per 4 consecutive output bytes of a row (row-major over frames x rows x 3W bytes).
__global__ void synth_kernel(int kind, uint64_t seed, const int64_t* __restrict__ frame_ids, int n_frames,
                             int H, int W, int64_t pitch, uint8_t* __restrict__ out) {
  const int64_t rowbytes = 3 * (int64_t)W;
  const int64_t words_per_row = (rowbytes + 3) / 4;
  const int64_t total = (int64_t)n_frames * H * words_per_row;
  const uint64_t s8 = (seed * 2654435761ull) & 0xFFull;
  const uint64_t smix = seed * 0xD1B54A32D192ED03ull;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < total; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = w / words_per_row, wc = w - row * words_per_row;
    const int64_t f = row / H, y = row - f * H;
    const int64_t fid = frame_ids[f];
    uint8_t* dst = out + f * H * pitch + y * pitch;
    for (int b = 0; b < 4; ++b) {
      const int64_t byte = wc * 4 + b;
      if (byte >= rowbytes) break;
      const int64_t x = byte / 3, c = byte - 3 * x;
      uint8_t v;
      if (kind == VP_SYNTH_RAMP) {
        v = (uint8_t)((s8 + (uint64_t)(fid * 97 + y * 31 + x * 7 + c)) & 0xFF);
      } else {
        const uint64_t lin = (uint64_t)(((fid * H + y) * W + x) * 3 + c);
        v = (uint8_t)(splitmix64(lin + smix) >> 56);
      }
      dst[byte] = v;
    }
  }
}

}  // namespace
}  // namespace vp

extern "C" vp_status vp_synth_frames(int32_t kind, uint64_t seed, const int64_t* frame_ids, int32_t n_frames,
                                     int32_t height, int32_t width, int64_t row_pitch, uint8_t* out, void* stream) {
  if (n_frames < 0 || height < 0 || width < 0 || row_pitch < 3 * (int64_t)width || (kind != 0 && kind != 1)) {
    vp::set_error("vp_synth_frames: invalid arguments");
    return VP_EINVAL;
  }
  if (n_frames == 0 || height == 0 || width == 0) return VP_OK;
  if (out == nullptr || frame_ids == nullptr) {
    vp::set_error("vp_synth_frames: null pointer argument");
    return VP_EINVAL;
  }
  vp::synth_kernel<<<148 * 8, 256, 0, vp::as_stream(stream)>>>(kind, seed, frame_ids, n_frames, height, width,
                                                                row_pitch, out);
  return vp::launch_status("vp_synth_frames");
}
