/*
 * vp.h -- C ABI of the B200 (sm_100a) visual-preprocessing hot path of EasyVideoR1
 * (arXiv 2604.16893).  The path: fps/max-frames frame sampling, smart_resize under separate
 * image/video budgets, antialiased bicubic resize, rescale + mean/std normalise,
 * temporal-patch/patch/spatial-merge patchify into Qwen-VL pixel_values + grid_thw, and
 * metadata-consistent 3D MRoPE position ids with strict placeholder validation.
 *
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n of the reference; O1-O11 / C1-C26 are the
 * steps / readings of SURVEY.md section 8(c), restated in DESIGN.md.
 *
 * Conventions for every entry point
 *   - All array arguments marked (dev) are device pointers owned by the caller; the library never
 *     allocates device memory (scratch is a caller-provided workspace) and keeps no state between calls
 *     beyond idempotent per-device caches (SM count, kernel shared-memory attributes), so calls are
 *     reentrant and thread-safe on any device and stream.
 *   - Work is enqueued on `stream` (a cudaStream_t, passed as void*; NULL = legacy default stream);
 *     no call synchronises the device, so every call is CUDA-graph capturable.
 *   - The return value reports host-detectable errors synchronously (null pointers, invalid
 *     parameters per S:31-33, unsupported sizes) and launch failures (VP_ECUDA).  It never waits for
 *     kernels.  Data-dependent errors (invalid clip descriptors S:79, placeholder mismatches
 *     P:165 / S:444, capacity overflow) are written to device status fields; the Python binding
 *     reads them and raises (strict by default).
 *   - vp_last_error_detail() returns a thread-local text of the last host-side error.
 *   - All integers are little-endian; structs are plain C with natural alignment (sizes asserted
 *     in the binding).
 */
#ifndef VP_H_
#define VP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VP_ABI_VERSION 1

typedef enum {
  VP_OK = 0,
  VP_EINVAL = 1,     /* invalid argument / invalid clip (total<=0 or fps<=0; h,w<1) */
  VP_EALIGN = 2,     /* misaligned pointer or pitch */
  VP_EMISMATCH = 3,  /* placeholder run length != t*h*w/m^2, or grids left over */
  VP_ECAPACITY = 4,  /* an output buffer is smaller than the plan requires */
  VP_ECUDA = 5,      /* kernel launch failed */
  VP_EUNSUPPORTED = 6 /* a configuration beyond the kernels' envelope (merge_size*patch_size > 64) */
} vp_status;

typedef enum { VP_SAMPLE_CENTER_BIN = 0 /* S:78 (C1, C2) */,
               VP_SAMPLE_LINSPACE = 1   /* HF Qwen3-VL sample_frames (C1/C2 HF rule, N1): n = int(total/src_fps*fps),
                                           clamped to [min_frames, min(max_frames, total)], no tp rounding;
                                           idx_i = round_half_even(i * (total-1)/(n-1)), idx_{n-1} = total-1 */
} vp_sampling;
typedef enum { VP_BUDGET_PER_FRAME = 0 /* P:271 */, VP_BUDGET_TOTAL = 1 /* Qwen3-VL T-aware, C8 */ } vp_budget_mode;
typedef enum { VP_ROPE_QWEN3_SPLIT = 0 /* C18 */, VP_ROPE_QWEN2 = 1 /* classic, C19 */,
               VP_ROPE_QWEN25 = 2 /* time-scaled, C19 */ } vp_rope_variant;
typedef enum { VP_OUT_BF16 = 0, VP_OUT_F32 = 1 } vp_dtype;
typedef enum { VP_RESIZE_FLOAT = 0 /* C11: float domain end to end, one clamp after the second pass */,
               VP_RESIZE_U8 = 1    /* N1 HF drop-in: torch's uint8 antialiased bicubic, bit-exact -- int16-precision
                                      coefficients (p = max bits with max|w|*2^p < 2^15), horizontal pass first,
                                      u8 (clamped, >> p with 2^(p-1) rounding) between and after the passes;
                                      downscales <= 15.5x per axis (else VP_EUNSUPPORTED) */ } vp_resize_mode;
typedef enum { VP_SYNTH_RAMP = 0 /* S:71 */, VP_SYNTH_NOISE = 1 } vp_synth_kind;

/* Preprocessing parameters (S:29-34 PreprocessParams; P:90 independent budgets; P:271 values).
 * Invariants checked on the host (VP_EINVAL): patch,merge,tp >= 1; max_frames >= tp;
 * video_max_pixels, image_max_pixels >= (patch*merge)^2; target_fps > 0; std[c] != 0; sampling in vp_sampling;
 * 0 <= min_frames <= max_frames; resize_mode in vp_resize_mode. */
typedef struct {
  double  target_fps;          /* 2.0 */
  int32_t max_frames;          /* 128 */
  int32_t temporal_patch_size; /* 2 */
  int32_t patch_size;          /* 16 (Qwen3-VL) */
  int32_t merge_size;          /* 2 */
  int64_t video_max_pixels;    /* 262144 per frame, or total n*H*W budget if budget_mode==TOTAL */
  int64_t image_max_pixels;    /* 1048576 */
  int64_t min_pixels;          /* 0 disables the upscale branch (C7) */
  int32_t budget_mode;         /* vp_budget_mode, videos only */
  int32_t sampling;            /* vp_sampling */
  double  mean[3];             /* per-channel mean (C13), 0.5 for Qwen3-VL */
  double  std[3];              /* per-channel std (C13), 0.5 for Qwen3-VL */
  int32_t out_dtype;           /* vp_dtype of pixel_values */
  int32_t launch_mask;         /* optional launch hint for vp_resize_normalize_patchify: totals[VP_TOT_VARIANTS]
                                  of the plan (bit v = some valid clip uses kernel variant v); kernels of absent
                                  variants are not launched.  0 = unknown: launch every kernel.  Ignored by the
                                  other calls.  A mask missing a present variant leaves its clips unwritten. */
  int32_t min_frames;          /* VP_SAMPLE_LINSPACE only: lower clamp of n (HF Qwen3-VL: 4) */
  int32_t resize_mode;         /* vp_resize_mode (plan and resize calls must agree) */
} vp_params;                   /* 120 bytes */

/* One input clip (S:42-47 VideoMetadata source fields).  Images: is_image=1, the frame count and
 * fps are ignored (an image is one frame, routed to the image budget and output, P:90 / P:165). */
typedef struct {
  int64_t total_source_frames;
  double  source_fps;
  int32_t height, width;       /* source frame size in pixels */
  int32_t is_image;
  int32_t pad_;
} vp_clip_desc;                /* 32 bytes */

/* Per-clip plan written by vp_plan_frames (O1-O3, H4).  Offsets are exclusive scans in clip order,
 * separately per modality (patch_offset, token_offset, grid_index, group_offset) or over all clips
 * (index_offset).  tile_* and kernel_variant are private to the library. */
typedef struct {
  int32_t status;              /* VP_OK or VP_EINVAL (such a clip produces no output) */
  int32_t is_image;
  int32_t in_h, in_w;          /* source size */
  int32_t n_frames;            /* sampled frames n (O1); 1 for images */
  int32_t out_h, out_w;        /* smart_resize result (O2) */
  int32_t grid_t, grid_h, grid_w; /* O3 */
  int64_t index_offset;        /* into frame_indices */
  int64_t patch_offset;        /* first row in this modality's pixel_values */
  int64_t token_offset;        /* first LLM token (t*h*w/m^2 units) within this modality */
  int64_t grid_index;          /* row in image_grid_thw / video_grid_thw */
  int64_t group_offset;        /* first entry of this video's group timestamps */
  int64_t tile_offset;         /* private */
  int32_t tile_count;          /* private */
  int32_t kernel_variant;      /* private */
  double  effective_fps;       /* n*src_fps/total (C23); 0 for images */
} vp_clip_plan;                /* 104 bytes */

/* Indices into the int64 totals[VP_TOT_LEN] array written by vp_plan_frames. */
enum {
  VP_TOT_INDICES = 0,   /* sum of n_frames over valid clips (entries needed in frame_indices) */
  VP_TOT_IMG_ROWS = 1,  /* rows of pixel_values (images) */
  VP_TOT_VID_ROWS = 2,  /* rows of pixel_values_videos */
  VP_TOT_IMG_TOKENS = 3,
  VP_TOT_VID_TOKENS = 4,
  VP_TOT_N_IMAGES = 5,
  VP_TOT_N_VIDEOS = 6,
  VP_TOT_VID_GROUPS = 7, /* sum of grid_t over videos (entries of group_timestamps) */
  VP_TOT_TILES = 8,      /* private */
  VP_TOT_FLAGS = 9,      /* bit0 frame_indices overflow, bit1 timestamps overflow */
  VP_TOT_N_INVALID = 10, /* clips with status != VP_OK */
  VP_TOT_VARIANTS = 11,  /* bitmask of the kernel variants of the valid clips (the vp_params.launch_mask hint) */
  VP_TOT_LEN = 12
};

/* ---------------------------------------------------------------------------------------------
 * vp_plan_frames -- H1-H4 + H9: frame plan, smart_resize, grid and offsets for n clips.
 *   O1: n = clamp(floor(total/src_fps*target_fps), tp, max_frames), n <= total (C3),
 *      rounded down to a multiple of tp; idx_i = min(total-1, floor((i+1/2)*total/n)).
 *      p->sampling == VP_SAMPLE_LINSPACE: the HF Qwen3-VL rule instead (see vp_sampling; a clip whose n is 0
 *      -- min_frames = 0 and a sub-frame duration -- is invalid).
 *   O2 (C5-C8): smart_resize under image_max_pixels (images) or video_max_pixels (videos,
 *      per-frame or total budget).  O3: grid = (ceil(n/tp), H'/p, W'/p).
 *   O10 (C22): per temporal group timestamp (idx[g*tp]/fps + idx[g*tp+tp-1]/fps)/2 after
 *      padding idx with its last entry.
 *   All f64 expressions are evaluated with IEEE round-to-nearest and no contraction, so every
 *   integer output is bit-identical to the oracle.
 * Args:
 *   p                 host pointer, parameters (validated on the host)
 *   clips (dev)       [n] clip descriptors
 *   n                 number of clips, 0 <= n
 *   plans (dev)       [n] output plans
 *   frame_indices (dev) [index_cap] int64 output; clip k's indices at plans[k].index_offset
 *   group_timestamps (dev, nullable) [ts_cap] f64 output; video v's groups at plans[v].group_offset
 *   totals (dev)      [VP_TOT_LEN] int64 output
 * Errors: VP_EINVAL (bad params / null pointers / n < 0), VP_ECUDA.  Invalid clips get
 *   plans[k].status = VP_EINVAL and contribute nothing; overflow of frame_indices / timestamps sets
 *   totals[VP_TOT_FLAGS] bits (entries beyond the caps are not written).
 * ------------------------------------------------------------------------------------------- */
vp_status vp_plan_frames(const vp_params* p, const vp_clip_desc* clips, int32_t n,
                         vp_clip_plan* plans, int64_t* frame_indices, int64_t index_cap,
                         double* group_timestamps, int64_t ts_cap, int64_t* totals, void* stream);

/* ---------------------------------------------------------------------------------------------
 * vp_resize_normalize_patchify -- H5-H7: fused AA-bicubic resize, clamp, rescale+normalise,
 * temporal pad and patchify (O4-O9) of every valid clip, plus grid_thw output.
 *   out[i][j][c] = clamp_[0,255]( sum_k wv[i,k] sum_l wh[j,l] src[y0_i+k][x0_j+l][c] )   (O4, O5)
 *   x = (out/255 - mean_c)/std_c (O6); frames n..tp*gt-1 repeat frame n-1 (O7);
 *   pixel_values[patch_offset + r][q] with r = (((t*(gh/m)+hb)*(gw/m)+wb)*m+mh)*m+mw,
 *   q = ((c*tp+ti)*p+py)*p+px (O8, HF layout P:78); stored as bf16 (RNE) or f32 (O9).
 * Args:
 *   p                  host pointer, same parameters as the plan call
 *   plans (dev)        [n] from vp_plan_frames (read only).  Any contiguous sub-range of one plan array
 *                      may be passed (plans + k0, n), e.g. to pipeline host->device copies clip by clip;
 *                      row offsets and grid indices stay those of the full batch.
 *   frames (dev)       u8 RGB, THWC.  Clip k's sampled frame f (f < n_frames; images f = 0) starts at
 *                      frames + clip_byte_offset[k] + f * in_h * row_pitch[k]; pixel (y,x,c) at
 *                      + y*row_pitch[k] + 3x + c.  row_pitch[k] >= 3*in_w.
 *   clip_byte_offset (dev) [n] int64;  row_pitch (dev) [n] int64
 *   pixel_values_images (dev, nullable if no images) [img_rows_cap, 3*tp*p*p] of out_dtype
 *   pixel_values_videos (dev, nullable if no videos) [vid_rows_cap, 3*tp*p*p] of out_dtype
 *   image_grid_thw, video_grid_thw (dev) [n_images,3] / [n_videos,3] int64 (HF convention)
 *   clip_status (dev, nullable) [n] int32 output: VP_OK, VP_EINVAL (invalid plan), VP_ECAPACITY
 *                      (rows beyond the cap; that clip's rows are not written) or VP_EUNSUPPORTED (VP_RESIZE_U8
 *                      beyond 15.5x; rows not written).  In VP_RESIZE_FLOAT mode every resize ratio is
 *                      supported (downscales beyond the shared-memory window tables, ~34x per axis, take a
 *                      direct f64 kernel)
 *   workspace (dev)    vp_resize_workspace_bytes(n) bytes, 256-B aligned, caller-owned scratch (work index and
 *                      per-clip weight tables, rebuilt on every call; contents need not persist)
 * Errors: VP_EINVAL (incl. a missing / short / misaligned workspace), VP_EUNSUPPORTED, VP_ECUDA.
 * ------------------------------------------------------------------------------------------- */
size_t vp_resize_workspace_bytes(int32_t n);
vp_status vp_resize_normalize_patchify(const vp_params* p, const vp_clip_plan* plans, int32_t n,
                                       const uint8_t* frames,
                                       const int64_t* clip_byte_offset, const int64_t* row_pitch,
                                       void* pixel_values_images, int64_t img_rows_cap,
                                       void* pixel_values_videos, int64_t vid_rows_cap,
                                       int64_t* image_grid_thw, int64_t* video_grid_thw,
                                       int32_t* clip_status, void* workspace, size_t workspace_bytes,
                                       void* stream);

/* ---------------------------------------------------------------------------------------------
 * vp_rope_index -- H8: 3D MRoPE position ids for a packed (padding-free) batch of B
 * sequences, with strict placeholder validation.  O11:
 *   per sequence, maximal runs of equal token type; p starts at 0.  Text run of length L:
 *   ids (p+j, p+j, p+j), p += L.  Visual run: the next grid of its modality in batch order
 *   (QWEN3_SPLIT expands each video into grid_t grids (1,h,w), C18); the run length must equal
 *   t*(h/m)*(w/m); ids over (ti,hi,wi) row-major are (p+ti*iv, p+hi, p+wi);
 *   p += max((t-1)*iv, h/m-1, w/m-1) + 1.  delta = max_id + 1 - len (C21).
 *   iv = 1 (QWEN2) or tokens_per_second*int(second_per_grid[v]) (QWEN25); unused for QWEN3_SPLIT.
 * Args:
 *   p                 host pointer (merge_size is used)
 *   mm_token_type (dev) [total_L] int8: 0 text, 1 image, 2 video
 *   cu_seqlens (dev)  [B+1] int64, cu_seqlens[0] = 0, non-decreasing, cu_seqlens[B] = total_L
 *   image_grid_thw / video_grid_thw (dev) [n_images,3] / [n_videos,3] int64
 *   second_per_grid (dev, nullable) [n_videos] f64, QWEN25 only
 *   position_ids (dev) [3, total_L] int64 output (axis-major)
 *   rope_deltas (dev) [B] int64 output
 *   seq_status (dev)  [B+1] int32 output: per sequence VP_OK / VP_EMISMATCH; entry B is the batch
 *                     status (VP_EMISMATCH if grids are left over or a run had no grid)
 *   workspace (dev)   vp_rope_index_workspace_bytes(B, n_videos) bytes, 16-B aligned
 * Errors: VP_EINVAL, VP_ECUDA.
 * ------------------------------------------------------------------------------------------- */
size_t vp_rope_index_workspace_bytes(int32_t B, int32_t n_videos);
vp_status vp_rope_index(const vp_params* p, int32_t variant, const int8_t* mm_token_type,
                        const int64_t* cu_seqlens, int32_t B, int64_t total_L,
                        const int64_t* image_grid_thw, int32_t n_images,
                        const int64_t* video_grid_thw, int32_t n_videos,
                        const double* second_per_grid, int32_t tokens_per_second,
                        int64_t* position_ids, int64_t* rope_deltas, int32_t* seq_status,
                        void* workspace, size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------------------------
 * vp_pack_offsets -- H10: after an all-gather of every rank's per-clip (t, h, w, tokens) int32
 * records (ranks in order, clips_per_rank records each), write the global exclusive scan of
 * tokens and of patches (t*h*w) for all world*clips_per_rank clips.  Used for micro-batch
 * packing (P:271 dynamic batching).  gathered (dev) [world*clips_per_rank*4] int32;
 * token_offsets, patch_offsets (dev) [world*clips_per_rank + 1] int64 (last = totals).
 * ------------------------------------------------------------------------------------------- */
vp_status vp_pack_offsets(const int32_t* gathered, int32_t world, int32_t clips_per_rank,
                          int64_t* token_offsets, int64_t* patch_offsets, void* stream);

/* Per-clip (t, h, w, tokens) int32 records of this rank's plans, for the all-gather of H10.
 * plans (dev) [n]; records (dev) [n*4].  Invalid clips give (0,0,0,0). */
vp_status vp_plan_records(const vp_clip_plan* plans, int32_t n, int32_t merge_size,
                          int32_t* records, void* stream);

/* ---------------------------------------------------------------------------------------------
 * vp_plan_second_per_grid -- N2 (Qwen2.5-VL time-scaled MRoPE, C19): per valid video, the seconds one temporal
 * grid spans, second_per_grid[grid_index] = temporal_patch_size / sampled_fps with HF's sampled fps
 * n / total * source_fps (evaluated in that f64 order, no contraction).  Feeds vp_rope_index(VP_ROPE_QWEN25).
 * clips (dev) [n], plans (dev) [n] of the same vp_plan_frames call; second_per_grid (dev) [n_videos] f64.
 * ------------------------------------------------------------------------------------------- */
vp_status vp_plan_second_per_grid(const vp_clip_desc* clips, const vp_clip_plan* plans, int32_t n,
                                  int32_t temporal_patch_size, double* second_per_grid, void* stream);

/* ---------------------------------------------------------------------------------------------
 * vp_dedup_clips -- N3: hash-based deduplication of a batch ("hash-based deduplication"; GRPO n = 8 rollouts
 * per prompt).  keys (dev) [n] uint64: one caller-chosen key per sample's clip (e.g. a hash of the video id
 * and the sampling parameters; the library does not hash frame bytes -- reading them costs as much as processing
 * them).  Outputs: unique_id (dev) [n] int32 = dense id of the sample's key in order of first occurrence;
 * unique_list (dev) [n] int32, first *n_unique entries = the batch index of each key's first occurrence, in batch
 * order; n_unique (dev) int32.  The caller plans and resizes clips[unique_list[0..U)] only.  One CTA; O(n^2 / 1024)
 * key compares per thread.  Errors: VP_EINVAL, VP_ECUDA.
 *
 * vp_dedup_views -- per sample, its view into the unique clips' outputs: patch_offset (dev) [n] int64 (first row
 * in the unique pixel_values of its modality; -1 if the clip is invalid), grid_thw (dev) [n,3] int64 (the sample's
 * grid, e.g. for vp_rope_index over every sample's sequence), status (dev, nullable) [n] int32 (plan status).
 * unique_plans (dev) [U] from vp_plan_frames over the unique clips; unique_id from vp_dedup_clips.
 * ------------------------------------------------------------------------------------------- */
vp_status vp_dedup_clips(const uint64_t* keys, int32_t n, int32_t* unique_id, int32_t* unique_list,
                         int32_t* n_unique, void* stream);
vp_status vp_dedup_views(const vp_clip_plan* unique_plans, const int32_t* unique_id, int32_t n,
                         int64_t* patch_offset, int64_t* grid_thw, int32_t* status, void* stream);

/* ---------------------------------------------------------------------------------------------
 * vp_nv12_to_rgb -- N4 upstream: NVDEC-style NV12 frames (Y plane, then an interleaved U,V plane of height/2 rows,
 * 4:2:0, each 2x2 block sharing one U,V pair) -> u8 RGB THWC, BT.601 limited range in OpenCV's fixed-point form
 * (COLOR_YUV2RGB_NV12): y' = max(0, Y-16)*1220542, R = sat((y' + 2^19 + 1673527*(V-128)) >> 20),
 * G = sat((y' + 2^19 - 852492*(V-128) - 409993*(U-128)) >> 20), B = sat((y' + 2^19 + 2116026*(U-128)) >> 20).
 * P:73 ("decodes, resamples, and resizes"): the decoder output feeds K3 without a host round trip.
 *   y, uv (dev): frame f's planes at y + f*frame_stride and uv + f*frame_stride, rows `pitch` bytes apart;
 *   rgb (dev): frame f row r at rgb + f*rgb_frame_stride + r*rgb_pitch (e.g. a clip's slot in the K3 frame buffer).
 *   height, width even, >= 2.  Errors: VP_EINVAL, VP_ECUDA.
 *
 * vp_vision_ids -- N4 downstream: for the vision tower, per pixel_values row (O8 order) of every grid in
 * grid_thw (dev) [n_grids,3]: pos_ids (dev) [sum t*h*w, 2] int32 = (hb*m + mh, wb*m + mw) (its patch's row and
 * column in the frame); cu_seqlens (dev) [sum t + 1] int32 = 0 then the cumulative patch count at the end of every
 * temporal patch (X: HF Qwen3-VL vision model rot_pos_emb and cu_seqlens).  workspace (dev)
 * vp_vision_ids_workspace_bytes(n_grids) bytes, 8-B aligned.  Errors: VP_EINVAL, VP_ECUDA.
 * ------------------------------------------------------------------------------------------- */
vp_status vp_nv12_to_rgb(const uint8_t* y, const uint8_t* uv, int64_t pitch, int64_t frame_stride, int32_t height,
                         int32_t width, int32_t n_frames, uint8_t* rgb, int64_t rgb_pitch, int64_t rgb_frame_stride,
                         void* stream);
size_t vp_vision_ids_workspace_bytes(int32_t n_grids);
vp_status vp_vision_ids(const int64_t* grid_thw, int32_t n_grids, int32_t merge_size, int32_t* pos_ids,
                        int32_t* cu_seqlens, void* workspace, size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------------------------
 * vp_synth_frames -- test/bench input generator (not part of the hot path; never timed).
 *   RAMP: (seed*2654435761 + i*97 + y*31 + x*7 + c) mod 256, i = frame_ids[f]
 *   NOISE : top 8 bits of splitmix64(((i*H + y)*W + x)*3 + c + seed*0xD1B54A32D192ED03)
 * Writes n_frames frames of height x width x 3 u8 at out + f*height*row_pitch (dev).
 * ------------------------------------------------------------------------------------------- */
vp_status vp_synth_frames(int32_t kind, uint64_t seed, const int64_t* frame_ids, int32_t n_frames,
                          int32_t height, int32_t width, int64_t row_pitch, uint8_t* out, void* stream);

const char* vp_status_string(vp_status s);
const char* vp_last_error_detail(void);
int32_t vp_abi_version(void);
/* sizeof checks for bindings: returns sizeof(vp_params), sizeof(vp_clip_desc), sizeof(vp_clip_plan)
 * packed as params | desc<<10 | plan<<20. */
int32_t vp_struct_sizes(void);

#ifdef __cplusplus
}
#endif
#endif /* VP_H_ */
