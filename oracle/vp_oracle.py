"""Plain, slow, f64 CPU oracle of the EasyVideoR1 visual-preprocessing hot path.

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs, never by the product package.  Shares no code,
tables or constants with the CUDA path.

Citations: ``P:n`` = PAPER.md line n, ``S:n`` = SPEC.md line n (both under the read-only
reference), ``O*``/``C*`` = the numbered steps / readings of SURVEY.md §8(c) (restated in
DESIGN.md §3).  Every function follows the paper's (or the chosen reading's) definition
step by step; library primitives (numpy matmul, reshape/transpose) serve only as whole
steps.  Python floats are IEEE binary64 and are never FMA-contracted, so every planning
expression below is evaluated exactly as written.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``): SPEC worked examples (tests/golden/),
closed-form bounds, HF transformers' ``smart_resize`` / processors / ``get_rope_index``,
torch's float64 antialiased bicubic, brute force on tiny inputs.  Parity unpinned (by a
library): the classic multi-t MRoPE variant (C19) beyond invariants and the HF docstring
example -- see DESIGN.md.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "VP_OK", "VP_EINVAL", "VP_EMISMATCH",
    "sample_frame_indices", "sample_frame_indices_hf", "effective_fps", "round_half_even_div", "smart_resize",
    "smart_resize_exact_floor", "grid_thw", "clip_budget", "plan_clip", "plan_batch",
    "keys_cubic", "aa_weights", "weight_matrix", "resize_frame", "resize_pixel",
    "normalize", "temporal_pad", "patchify", "patch_coords", "bf16_rne_bits", "bf16_bits_to_f64",
    "group_timestamps", "hf_sampled_fps", "second_per_grid", "qwen25_interval", "rope_index", "process_batch", "ClipPlan",
    "dedup_keys", "quantize_weights_u8", "resize_frame_u8", "nv12_to_rgb", "vision_pos_ids", "vision_cu_seqlens",
]

VP_OK, VP_EINVAL, VP_EMISMATCH = 0, 1, 3


# ---------------------------------------------------------------------------
# O1 -- frame plan.  S:75-83 (sample_frame_indices), "resamples", "2 FPS ... 128 frames"
# ---------------------------------------------------------------------------

def sample_frame_indices(total: int, src_fps: float, target_fps: float, max_frames: int, tp: int):
    """Center-of-bin frame indices with reading C3 (n never exceeds total).

    d   = floor((total / src_fps) * target_fps)           (f64, as S:78 "floor(dur*fps)")
    n   = min(max(d, tp), max_frames); n = min(n, total)  (clamp, C3)
    n   = tp * (n div tp) if n >= tp                      (round down to a multiple of tp)
    idx = min(total-1, floor((i + 1/2) * total / n))      (exact integer form (2i+1)*total div 2n)
    Returns (n, [idx...]).  Raises ValueError on total<1 or fps<=0.
    """
    if total < 1 or not (src_fps > 0):
        raise ValueError("invalid input: total_source_frames >= 1 and source_fps > 0 required (S:79)")
    d = math.floor((float(total) / float(src_fps)) * float(target_fps))
    n = min(max(d, tp), max_frames)
    n = min(n, total)
    if n >= tp:
        n = tp * (n // tp)
    idx = [min(total - 1, ((2 * i + 1) * total) // (2 * n)) for i in range(n)]
    return n, idx


def sample_frame_indices_hf(total: int, src_fps: float, target_fps: float, min_frames: int, max_frames: int):
    """HF drop-in sampling (reading C1/C2, HF rule; N1): Qwen3-VL's ``sample_frames``.

    n   = int(total / src_fps * target_fps)                 (f64, truncation)
    n   = min(max(n, min_frames), max_frames, total)       (no rounding to a multiple of tp)
    idx = round_half_even(linspace(0, total - 1, n))      (numpy linspace: i * ((total-1)/(n-1)), last = total-1)
    Returns (n, [idx...]).  Raises ValueError on total<1, fps<=0 or n == 0."""
    if total < 1 or not (src_fps > 0):
        raise ValueError("invalid input: total_source_frames >= 1 and source_fps > 0 required (S:79)")
    n = int(float(total) / float(src_fps) * float(target_fps))
    n = min(max(n, min_frames), max_frames, total)
    if n < 1:
        raise ValueError("no frame sampled")
    if n == 1:
        return 1, [0]
    step = float(total - 1) / float(n - 1)
    idx = [round(i * step) for i in range(n - 1)] + [total - 1]     # Python round: half to even
    return n, idx


def effective_fps(n: int, src_fps: float, total: int) -> float:
    """C23: effective fps of the sampled sequence = n * src_fps / total (S:44 names it, no formula)."""
    return (float(n) * float(src_fps)) / float(total)


# ---------------------------------------------------------------------------
# O2 -- smart_resize.  S:85-93; P:90 independent budgets; readings C5-C9
# ---------------------------------------------------------------------------

def round_half_even_div(a: int, f: int) -> int:
    """rne(a / f) for non-negative integers, in integers (C5: Python round() semantics)."""
    q, r = divmod(a, f)
    if 2 * r > f or (2 * r == f and q % 2 == 1):
        q += 1
    return q


def smart_resize(h: int, w: int, budget: int, factor: int, min_pixels: int = 0,
                 n_frames: int | None = None, tp: int = 1):
    """(H', W') multiples of ``factor`` under ``budget``.

    Per-frame mode (n_frames None):   area = hb*wb,        scale term = h*w        (C6)
    Total mode (n_frames = n, C8):    area = tb*hb*wb,     scale term = n*h*w, tb = ceil(n/tp)*tp
      hb = max(f, f*rne(h/f)); wb likewise                                   (S:88 + C5)
      if area > budget:  beta = sqrt(term/budget); hb = max(f, floor(h/beta/f)*f)   (C6, f64)
      elif min_pixels>0 and area < min_pixels: beta = sqrt(min_pixels/term);
                         hb = ceil(h*beta/f)*f                                (C7)
    """
    f = factor
    hb = max(f, f * round_half_even_div(h, f))
    wb = max(f, f * round_half_even_div(w, f))
    if n_frames is None:
        area, term = hb * wb, h * w
    else:
        tb = -(-n_frames // tp) * tp
        area, term = tb * hb * wb, n_frames * h * w
    if area > budget:
        beta = math.sqrt(float(term) / float(budget))
        hb = max(f, math.floor(float(h) / beta / float(f)) * f)
        wb = max(f, math.floor(float(w) / beta / float(f)) * f)
    elif min_pixels > 0 and area < min_pixels:
        beta = math.sqrt(float(min_pixels) / float(term))
        hb = math.ceil(float(h) * beta / float(f)) * f
        wb = math.ceil(float(w) * beta / float(f)) * f
    return hb, wb


def smart_resize_exact_floor(h: int, w: int, budget: int, factor: int):
    """Exact-integer version of the scaled branch (per-frame mode), used as a cross-check of C6:
    the largest k with (k*f)^2 * w <= h * budget  (i.e. k*f <= h*sqrt(b/(h*w))), floored at f."""
    def largest(a, other):
        # largest k >= 0 with (k f)^2 * other <= a * budget
        k = math.isqrt((a * budget) // (other * factor * factor))
        while ((k + 1) * factor) ** 2 * other <= a * budget:
            k += 1
        while k > 0 and (k * factor) ** 2 * other > a * budget:
            k -= 1
        return max(factor, k * factor)
    return largest(h, w), largest(w, h)


# ---------------------------------------------------------------------------
# O3 -- grid_thw.
# ---------------------------------------------------------------------------

def grid_thw(n: int, H: int, W: int, p: int, tp: int):
    """(ceil(T/tp), H/p, W/p); raises on non-divisible H or W (S:99 alignment error)."""
    if H % p or W % p:
        raise ValueError("alignment error: H and W must be divisible by patch_size (S:99)")
    return (-(-n // tp), H // p, W // p)


# ---------------------------------------------------------------------------
# Whole-clip plan (O1-O3 + routing by modality, P:90 / P:165)
# ---------------------------------------------------------------------------

@dataclass
class ClipPlan:
    status: int
    is_image: bool
    n: int = 0
    idx: list = field(default_factory=list)
    in_h: int = 0
    in_w: int = 0
    out_h: int = 0
    out_w: int = 0
    grid: tuple = (0, 0, 0)
    patches: int = 0
    tokens: int = 0
    eff_fps: float = 0.0
    # offsets filled by plan_batch (H4): per-modality exclusive scans in clip order
    index_offset: int = 0
    patch_offset: int = 0
    token_offset: int = 0
    grid_index: int = 0
    group_offset: int = 0


def clip_budget(params: dict, is_image: bool) -> int:
    """images use image_max_pixels, videos video_max_pixels (independent budgets)."""
    return int(params["image_max_pixels"] if is_image else params["video_max_pixels"])


def plan_clip(params: dict, c: dict) -> ClipPlan:
    tp, p, m = params["temporal_patch_size"], params["patch_size"], params["merge_size"]
    f = p * m
    is_image = bool(c["is_image"])
    h, w = int(c["height"]), int(c["width"])
    if h < 1 or w < 1:
        return ClipPlan(VP_EINVAL, is_image)
    if is_image:                     # an image is one frame, index 0 (O1 images)
        n, idx, eff = 1, [0], 0.0
        H, W = smart_resize(h, w, clip_budget(params, True), f, params["min_pixels"])
    else:
        try:
            if params.get("sampling", 0) == 1:
                n, idx = sample_frame_indices_hf(int(c["total_source_frames"]), float(c["source_fps"]),
                                                 float(params["target_fps"]), int(params.get("min_frames", 4)),
                                                 int(params["max_frames"]))
            else:
                n, idx = sample_frame_indices(int(c["total_source_frames"]), float(c["source_fps"]),
                                              float(params["target_fps"]), int(params["max_frames"]), tp)
        except ValueError:
            return ClipPlan(VP_EINVAL, is_image)
        eff = effective_fps(n, float(c["source_fps"]), int(c["total_source_frames"]))
        if params["budget_mode"] == 1:
            H, W = smart_resize(h, w, clip_budget(params, False), f, params["min_pixels"], n_frames=n, tp=tp)
        else:
            H, W = smart_resize(h, w, clip_budget(params, False), f, params["min_pixels"])
    g = grid_thw(n, H, W, p, tp)
    patches = g[0] * g[1] * g[2]
    return ClipPlan(VP_OK, is_image, n, idx, h, w, H, W, g, patches, patches // (m * m), eff)


def plan_batch(params: dict, clips):
    """H4: per-modality exclusive scans (clip order) of patch rows, tokens, grid ordinals and
    video temporal groups; frame-index offsets over all clips.  Returns (plans, totals dict)."""
    plans = [plan_clip(params, c) for c in clips]
    tot = dict(indices=0, img_rows=0, vid_rows=0, img_tokens=0, vid_tokens=0, n_images=0, n_videos=0,
               vid_groups=0)
    for pl in plans:
        pl.index_offset = tot["indices"]
        tot["indices"] += pl.n
        if pl.status != VP_OK:
            continue
        if pl.is_image:
            pl.patch_offset, pl.token_offset, pl.grid_index = tot["img_rows"], tot["img_tokens"], tot["n_images"]
            tot["img_rows"] += pl.patches
            tot["img_tokens"] += pl.tokens
            tot["n_images"] += 1
        else:
            pl.patch_offset, pl.token_offset, pl.grid_index = tot["vid_rows"], tot["vid_tokens"], tot["n_videos"]
            pl.group_offset = tot["vid_groups"]
            tot["vid_rows"] += pl.patches
            tot["vid_tokens"] += pl.tokens
            tot["n_videos"] += 1
            tot["vid_groups"] += pl.grid[0]
    return plans, tot


# ---------------------------------------------------------------------------
# O4 -- antialiased bicubic weights (reading C10: PIL / torch-AA semantics, Keys a = -0.5)
# ---------------------------------------------------------------------------

def keys_cubic(x: float, a: float = -0.5) -> float:
    """Keys cubic convolution kernel (a = -0.5)."""
    x = abs(x)
    if x < 1.0:
        return ((a + 2.0) * x - (a + 3.0)) * x * x + 1.0
    if x < 2.0:
        return (((x - 5.0) * x + 8.0) * x - 4.0) * a
    return 0.0


def aa_weights(in_size: int, out_size: int):
    """Per output index i: (x0, w[0..len)) with
       scale = in/out, fs = max(scale, 1), support = 2*fs, c = (i + 0.5)*scale,
       x0 = max(0, int(c - support + 0.5)), x1 = min(in, int(c + support + 0.5)),
       w_k = K((k + x0 - c + 0.5) * (1/fs)) normalised by their sum.   (C10)"""
    scale = float(in_size) / float(out_size)
    fs = max(scale, 1.0)
    support = 2.0 * fs
    inv = 1.0 / fs
    out = []
    for i in range(out_size):
        c = (i + 0.5) * scale
        x0 = max(0, int(c - support + 0.5))
        x1 = min(in_size, int(c + support + 0.5))
        w = np.array([keys_cubic((k + x0 - c + 0.5) * inv) for k in range(x1 - x0)], dtype=np.float64)
        s = w.sum()
        out.append((x0, w / s if s != 0.0 else w))
    return out


def quantize_weights_u8(in_size: int, out_size: int):
    """N1 (HF drop-in: HF resizes uint8 frames on torch's uint8 antialiased path, reading C11): the aa_weights of an
    axis as int16 fixed-point coefficients.  Precision p = the largest p <= 22 with max|w| * 2^(p+1) >= 2^15 not yet
    reached, i.e. max|w| * 2^p < 2^15; c = w * 2^p rounded half away from zero.  Returns ([(x0, [c...])], p)."""
    # the C10 window and weights, normalised with a sequential sum (as the integer path sums them; a last-ulp
    # difference could flip a coefficient's rounding)
    scale = float(in_size) / float(out_size)
    fs = max(scale, 1.0)
    ws = []
    for i in range(out_size):
        c = (i + 0.5) * scale
        x0 = max(0, int(c - 2.0 * fs + 0.5))
        x1 = min(in_size, int(c + 2.0 * fs + 0.5))
        w = [keys_cubic((k + x0 - c + 0.5) * (1.0 / fs)) for k in range(x1 - x0)]
        tot = 0.0
        for v in w:
            tot += v
        ws.append((x0, [v / tot for v in w] if tot != 0.0 else w))
    mx = max(max(abs(v) for v in w) for _, w in ws)
    p = 0
    while p < 22 and mx * float(1 << (p + 1)) < float(1 << 15):
        p += 1
    q = []
    for x0, w in ws:
        q.append((x0, [int(v * (1 << p) + 0.5) if v >= 0 else int(v * (1 << p) - 0.5) for v in w]))
    return q, p


def resize_frame_u8(frame_u8: np.ndarray, out_h: int, out_w: int) -> np.ndarray:
    """N1: separable AA bicubic in integers, horizontal pass first (when out_w != W), then vertical (when
    out_h != H); each pass: acc = 2^(p-1) + sum_k c_k * x_k, out = clamp(acc >> p, 0, 255) as u8 (so the
    intermediate is quantised, unlike O5).  frame_u8 [H, W, 3] -> u8 [out_h, out_w, 3]."""
    x = frame_u8.astype(np.int64)
    H, W, _ = x.shape
    if out_w != W:
        q, p = quantize_weights_u8(W, out_w)
        y = np.zeros((H, out_w, 3), dtype=np.int64)
        for j, (x0, c) in enumerate(q):
            acc = np.full((H, 3), 1 << (p - 1), dtype=np.int64)
            for k, ck in enumerate(c):
                acc += ck * x[:, x0 + k, :]
            y[:, j, :] = np.clip(acc >> p, 0, 255)
        x = y
    if out_h != H:
        q, p = quantize_weights_u8(H, out_h)
        y = np.zeros((out_h, x.shape[1], 3), dtype=np.int64)
        for i, (y0, c) in enumerate(q):
            acc = np.full((x.shape[1], 3), 1 << (p - 1), dtype=np.int64)
            for k, ck in enumerate(c):
                acc += ck * x[y0 + k, :, :]
            y[i] = np.clip(acc >> p, 0, 255)
        x = y
    return x.astype(np.uint8)


def weight_matrix(in_size: int, out_size: int) -> np.ndarray:
    """Dense [out, in] operator of aa_weights (zeros outside each window)."""
    M = np.zeros((out_size, in_size), dtype=np.float64)
    for i, (x0, w) in enumerate(aa_weights(in_size, out_size)):
        M[i, x0:x0 + len(w)] = w
    return M


# ---------------------------------------------------------------------------
# O5 -- separable resize, float domain end to end, clamp once after the second pass (C11, C12)
# ---------------------------------------------------------------------------

def resize_frame(frame_u8: np.ndarray, out_h: int, out_w: int) -> np.ndarray:
    """frame (H, W, 3) u8 -> (out_h, out_w, 3) f64 in [0, 255].
    tmp[y][j] = sum_k wh[j,k] src[y][x0_j+k]   (horizontal pass)
    out[i][j] = sum_k wv[i,k] tmp[y0_i+k][j]   (vertical pass), then clamp to [0, 255]."""
    H, W, _ = frame_u8.shape
    src = frame_u8.astype(np.float64)
    Wh = weight_matrix(W, out_w)           # [out_w, W]
    Wv = weight_matrix(H, out_h)           # [out_h, H]
    out = np.empty((out_h, out_w, 3), dtype=np.float64)
    for c in range(3):
        tmp = src[:, :, c] @ Wh.T          # [H, out_w]
        out[:, :, c] = Wv @ tmp            # [out_h, out_w]
    return np.clip(out, 0.0, 255.0)


def resize_pixel(frame_u8: np.ndarray, out_h: int, out_w: int, i: int, j: int, c: int,
                 _cache: dict | None = None) -> float:
    """One output value of resize_frame computed on its own (for sampled checks at full size):
    out[i][j][c] = clamp(sum_k wv[i,k] * (sum_l wh[j,l] * src[y0+k][x0+l][c]))."""
    H, W, _ = frame_u8.shape
    key = (H, W, out_h, out_w)
    if _cache is not None and key in _cache:
        wv_all, wh_all = _cache[key]
    else:
        wv_all, wh_all = aa_weights(H, out_h), aa_weights(W, out_w)
        if _cache is not None:
            _cache[key] = (wv_all, wh_all)
    y0, wv = wv_all[i]
    x0, wh = wh_all[j]
    block = frame_u8[y0:y0 + len(wv), x0:x0 + len(wh), c].astype(np.float64)
    tmp = block @ wh                         # horizontal pass for the rows in the window
    v = float(wv @ tmp)                      # vertical pass
    return min(max(v, 0.0), 255.0)


# ---------------------------------------------------------------------------
# O6-O9 -- normalise, temporal pad, patchify, output dtype
# ---------------------------------------------------------------------------

def normalize(x: np.ndarray, mean, std) -> np.ndarray:
    """O6 / C14: ((v / 255) - mean_c) / std_c in f64, channel last."""
    mean = np.asarray(mean, dtype=np.float64)
    std = np.asarray(std, dtype=np.float64)
    return (x / 255.0 - mean) / std


def temporal_pad(frames: np.ndarray, tp: int) -> np.ndarray:
    """O7 / C16: frames n .. tp*ceil(n/tp)-1 are copies of frame n-1 (an image becomes tp frames)."""
    n = frames.shape[0]
    pad = (-n) % tp
    if pad:
        frames = np.concatenate([frames, np.repeat(frames[-1:], pad, axis=0)], axis=0)
    return frames


def patchify(frames: np.ndarray, p: int, m: int, tp: int) -> np.ndarray:
    """O8 / C17: (T, H, W, 3) -> [gt*gh*gw, 3*tp*p*p] with
       row r = (((t*(gh/m) + hb)*(gw/m) + wb)*m + mh)*m + mw,
       col q = ((c*tp + ti)*p + py)*p + px,
       value = x[t*tp+ti][(hb*m+mh)*p+py][(wb*m+mw)*p+px][c]."""
    x = temporal_pad(frames, tp)
    T, H, W, C = x.shape
    gt, gh, gw = T // tp, H // p, W // p
    v = x.reshape(gt, tp, gh // m, m, p, gw // m, m, p, C)
    #            0   1   2      3  4  5      6  7  8
    # row (t, hb, wb, mh, mw), col (c, ti, py, px)
    v = v.transpose(0, 2, 5, 3, 6, 8, 1, 4, 7)
    return v.reshape(gt * gh * gw, C * tp * p * p)


def patch_coords(r: int, q: int, grid, p: int, m: int, tp: int):
    """Inverse of O8 for one element: (frame slot t*tp+ti, y, x, c) of pixel_values[r, q]."""
    gt, gh, gw = grid
    mw = r % m; r //= m
    mh = r % m; r //= m
    wb = r % (gw // m); r //= (gw // m)
    hb = r % (gh // m); t = r // (gh // m)
    px = q % p; q //= p
    py = q % p; q //= p
    ti = q % tp; c = q // tp
    return t * tp + ti, (hb * m + mh) * p + py, (wb * m + mw) * p + px, c


def bf16_rne_bits(x) -> np.ndarray:
    """O9 / C15: round each f64 value directly to the nearest bfloat16 (ties to even mantissa);
    returns the uint16 bit patterns.  No intermediate rounding to float32."""
    x = np.asarray(x, dtype=np.float64)
    mant, ex = np.frexp(x)                     # x = mant * 2**ex, |mant| in [0.5, 1)
    q = np.rint(mant * 256.0)                  # 8 significant bits; rint = half-to-even
    y = np.ldexp(q / 256.0, ex)                # exactly representable in bf16 (and f32)
    return (y.astype(np.float32).view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def bf16_bits_to_f64(bits) -> np.ndarray:
    b = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)
    return b.view(np.float32).astype(np.float64)


# ---------------------------------------------------------------------------
# O10 -- per temporal-group timestamps (reading C22)
# ---------------------------------------------------------------------------

def group_timestamps(idx, src_fps: float, tp: int):
    """Pad idx by repeating its last entry to a multiple of tp; ts_g = (idx[g*tp]/fps + idx[g*tp+tp-1]/fps)/2."""
    idx = list(idx)
    if len(idx) % tp:
        idx += [idx[-1]] * (tp - len(idx) % tp)
    ts = [i / float(src_fps) for i in idx]
    return [(ts[g] + ts[g + tp - 1]) / 2 for g in range(0, len(ts), tp)]


# ---------------------------------------------------------------------------
# O11 -- MRoPE position ids + strict placeholder validation (C18-C24)
# ---------------------------------------------------------------------------

def hf_sampled_fps(n: int, total: int, src_fps: float) -> float:
    """HF VideoMetadata.sampled_fps: len(indices) / total_num_frames * fps (f64, in this order)."""
    return n / float(total) * float(src_fps)


def second_per_grid(tp: int, sampled_fps: float) -> float:
    """Seconds spanned by one temporal grid of a video (Qwen2.5-VL, reading C19): tp / sampled fps
    (X: HF Qwen2_5_VLProcessor, ``second_per_grid_ts = temporal_patch_size / fps``); the sampled fps is the
    effective fps of O1 (C23)."""
    return tp / float(sampled_fps)


def qwen25_interval(tokens_per_second: int, second_per_grid_t: float) -> int:
    """Temporal id step between consecutive grids of one video (QWEN25 time-scaled MRoPE, C19):
    tokens_per_second * int(second_per_grid_t) -- int() truncates toward zero (X: HF Qwen2.5-VL
    ``get_rope_index``: ``time_interval = tokens_per_second * int(second_per_grid_t)``; its docstring:
    tps 25, tp 2, fps 1 -> interval 50)."""
    return int(tokens_per_second) * int(second_per_grid_t)


def rope_index(seqs, image_grids, video_grids, merge: int, variant: int = 0, second_per_grid_ts=None,
               tokens_per_second: int = 0):
    """seqs: list of 1-D int arrays of token types (0 text, 1 image, 2 video), one per sequence.
    image_grids / video_grids: lists of (t, h, w) in order of appearance across the batch.
    variant 0 (QWEN3_SPLIT): each video (t,h,w) is consumed as t grids (1,h,w) (C18).
    variant 1 (QWEN2 classic): temporal id p + ti (C19).
    variant 2 (QWEN25 time-scaled): temporal id p + ti*iv_v, iv_v = qwen25_interval(tokens_per_second,
    second_per_grid_ts[v]) (C19).
    Returns (ids list of int64 [3, L] arrays, deltas list, seq_status list, batch_status).
    A visual run whose length != t*(h/m)*(w/m), or with no grid left, is VP_EMISMATCH (C24);
    grids left unused at the end of the batch make batch_status VP_EMISMATCH."""
    img = [tuple(int(v) for v in g) + (1,) for g in image_grids]
    vid = []
    for v, g in enumerate(video_grids):
        t, h, w = (int(x) for x in g)
        iv = qwen25_interval(tokens_per_second, second_per_grid_ts[v]) if variant == 2 else 1
        vid += [(1, h, w, 1)] * t if variant == 0 else [(t, h, w, iv)]
    grids = {1: img, 2: vid}
    used = {1: 0, 2: 0}
    all_ids, deltas, status = [], [], []
    for s in seqs:
        s = np.asarray(s).astype(np.int64)
        L = len(s)
        ids = np.zeros((3, L), dtype=np.int64)
        st = VP_OK
        p = 0
        k = 0
        while k < L:                               # maximal runs of equal token type
            e = k
            while e < L and s[e] == s[k]:
                e += 1
            typ, n = int(s[k]), e - k
            if typ == 0:
                ids[:, k:e] = p + np.arange(n)
                p += n
            else:
                if used[typ] >= len(grids[typ]):
                    st = VP_EMISMATCH
                    used[typ] += 1
                    k = e
                    continue
                t, h, w, iv = grids[typ][used[typ]]
                used[typ] += 1
                hh, ww = h // merge, w // merge
                if n != t * hh * ww:
                    st = VP_EMISMATCH
                for j in range(min(n, t * hh * ww)):
                    ti, hi, wi = j // (hh * ww), (j // ww) % hh, j % ww
                    ids[0, k + j] = p + ti * iv
                    ids[1, k + j] = p + hi
                    ids[2, k + j] = p + wi
                p += max((t - 1) * iv, hh - 1, ww - 1) + 1
            k = e
        all_ids.append(ids)
        deltas.append(int(ids.max()) + 1 - L if L > 0 else 0)
        status.append(st)
    batch = VP_OK if used[1] == len(img) and used[2] == len(vid) else VP_EMISMATCH
    return all_ids, deltas, status, batch


# ---------------------------------------------------------------------------
# Whole path for a batch of clips (H1-H7)
# ---------------------------------------------------------------------------

def process_batch(params: dict, clips, frames_list, plans=None):
    """frames_list[k]: u8 (n_k, H, W, 3) holding clip k's sampled frames (images: 1 frame).
    Returns dict(pixel_values_images, pixel_values_videos (f64), image_grid_thw, video_grid_thw,
    plans, totals)."""
    if plans is None:
        plans, totals = plan_batch(params, clips)
    else:
        totals = None
    p, m, tp = params["patch_size"], params["merge_size"], params["temporal_patch_size"]
    img_rows, vid_rows, img_grids, vid_grids = [], [], [], []
    for pl, fr in zip(plans, frames_list):
        if pl.status != VP_OK:
            continue
        if params.get("resize_mode", 0) == 1:        # N1: u8-quantised resize (torch uint8 AA path)
            res = np.stack([resize_frame_u8(fr[k], pl.out_h, pl.out_w) for k in range(pl.n)]).astype(np.float64)
        else:
            res = np.stack([resize_frame(fr[k], pl.out_h, pl.out_w) for k in range(pl.n)])
        xn = normalize(res, params["mean"], params["std"])
        rows = patchify(xn, p, m, tp)
        (img_rows if pl.is_image else vid_rows).append(rows)
        (img_grids if pl.is_image else vid_grids).append(pl.grid)
    D = 3 * tp * p * p
    cat = lambda L: np.concatenate(L) if L else np.zeros((0, D))
    return dict(pixel_values_images=cat(img_rows), pixel_values_videos=cat(vid_rows),
                image_grid_thw=np.array(img_grids, dtype=np.int64).reshape(-1, 3),
                video_grid_thw=np.array(vid_grids, dtype=np.int64).reshape(-1, 3),
                plans=plans, totals=totals)


# ---------------------------------------------------------------------------
# N3 -- hash-based deduplication of a batch ("hash-based deduplication"; GRPO n rollouts per prompt)
# ---------------------------------------------------------------------------

def dedup_keys(keys):
    """Keep the first occurrence of each key.  Returns (unique_id per sample = rank of its key's first occurrence
    among first occurrences, unique_list = batch indices of the first occurrences in batch order)."""
    first = {}
    unique_list, unique_id = [], []
    for k, key in enumerate(keys):
        if key not in first:
            first[key] = len(unique_list)
            unique_list.append(k)
        unique_id.append(first[key])
    return unique_id, unique_list


# ---------------------------------------------------------------------------
# N4 -- adjacent steps: NVDEC NV12 -> RGB upstream, vision-tower patch ids downstream
# ---------------------------------------------------------------------------

def nv12_to_rgb(y_plane: np.ndarray, uv_plane: np.ndarray) -> np.ndarray:
    """BT.601 limited-range YCbCr -> RGB in OpenCV's fixed-point form (COLOR_YUV2RGB_NV12; coefficients x 2^20:
    1.164 -> 1220542, 1.596 -> 1673527, -0.813 -> -852492, -0.391 -> -409993, 2.018 -> 2116026), chroma shared by
    each 2x2 block.  y_plane u8 [H, W], uv_plane u8 [H/2, W] (U, V interleaved).  Plain integer loops per pixel."""
    H, W = y_plane.shape
    out = np.zeros((H, W, 3), dtype=np.uint8)
    sat = lambda v: 0 if v < 0 else (255 if v > 255 else v)
    for r in range(H):
        for c in range(W):
            u = int(uv_plane[r // 2, 2 * (c // 2)]) - 128
            v = int(uv_plane[r // 2, 2 * (c // 2) + 1]) - 128
            yy = max(0, int(y_plane[r, c]) - 16) * 1220542
            half = 1 << 19
            out[r, c, 0] = sat((yy + half + 1673527 * v) >> 20)
            out[r, c, 1] = sat((yy + half - 852492 * v - 409993 * u) >> 20)
            out[r, c, 2] = sat((yy + half + 2116026 * u) >> 20)
    return out


def vision_pos_ids(grids, merge: int) -> np.ndarray:
    """Per pixel_values row of every (t, h, w) grid (O8 order: frame, merge-row block, merge-column block, mh, mw),
    the patch's (row, col) in its frame: (hb*m + mh, wb*m + mw)  (X: HF Qwen3-VL vision rot_pos_emb)."""
    ids = []
    for t, h, w in grids:
        for _ in range(t):
            for hb in range(h // merge):
                for wb in range(w // merge):
                    for mh in range(merge):
                        for mw in range(merge):
                            ids.append((hb * merge + mh, wb * merge + mw))
    return np.array(ids, dtype=np.int64).reshape(-1, 2)


def vision_cu_seqlens(grids) -> list:
    """0, then the cumulative patch count at the end of every temporal patch (frame) of every grid."""
    cu = [0]
    for t, h, w in grids:
        for _ in range(t):
            cu.append(cu[-1] + h * w)
    return cu
