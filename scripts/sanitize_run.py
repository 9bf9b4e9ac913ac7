"""Small invocations of every kernel of libvp for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
the cfg1 clip, a mixed batch that takes every K3 variant (copy, team, wide, fast mild/medium, generic, direct,
unaligned pitch -> generic), f32 and bf16, small launches (row-band team items) and a 300-clip launch (whole-frame
team items), K4 on the matching token sequences, and the H10 records/pack kernels."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch

import paper_2604_16893_b200 as vp
import vp_inputs as I
import oracle as O
from parity import host_frames, oracle_params, pack_frames


def one(pre, clips, pad=None):
    pl = pre.plan(clips)
    oplans, _ = O.plan_batch(oracle_params(pre.params), clips)
    fl = host_frames(oplans)
    pitches = [(3 * c["width"] + 15) // 16 * 16 if pad is None else 3 * c["width"] + pad for c in clips]
    buf, offs, pit = pack_frames(fl, pitches)
    out = pre.run(pl, buf, offs, pit, strict=False)
    m = pre.params.merge_size
    seqs = []
    for o in oplans:
        if o.status != O.VP_OK:
            continue
        if o.is_image:
            seqs.append(I.token_types([(0, 3), (1, o.tokens), (0, 2)]))
        else:
            runs = [(0, 4)]
            for _ in range(o.grid[0]):
                runs += [(0, 7), (2, o.grid[1] * o.grid[2] // m ** 2), (0, 1)]
            seqs.append(I.token_types(runs))
    tt = torch.from_numpy(np.concatenate(seqs)).cuda()
    cu = torch.tensor(np.concatenate([[0], np.cumsum([len(s) for s in seqs])]), dtype=torch.int64).cuda()
    pre.rope_index(tt, cu, out["image_grid_thw"], out["video_grid_thw"], strict=False)
    rec = torch.empty(pl.n * 4, dtype=torch.int32, device="cuda")
    vp.plan_records(pl.plans_dev, pl.n, m, rec)
    tok = torch.empty(pl.n + 1, dtype=torch.int64, device="cuda")
    pat = torch.empty(pl.n + 1, dtype=torch.int64, device="cuda")
    vp.pack_offsets(rec, 1, pl.n, tok, pat)
    torch.cuda.synchronize()


which = sys.argv[1] if len(sys.argv) > 1 else "all"
for dtype in (0, 1):
    params, c1 = I.config("cfg1")
    params["out_dtype"] = dtype
    one(vp.VisualPreprocessor(**params), c1)
    pre = vp.VisualPreprocessor(max_frames=5, video_max_pixels=32768, image_max_pixels=65536, out_dtype=dtype)
    mixed = [I.clip(9, 2.0, 250, 500), I.clip(7, 2.0, 720, 1280), I.image(64, 96), I.image(150, 40),
             I.image(1000, 1010), I.clip(3, 1.0, 20, 30), I.clip(0, 30.0, 64, 64), I.image(820, 1000)]
    one(pre, mixed)
    one(pre, mixed, pad=1)
    big = vp.VisualPreprocessor(image_max_pixels=1024, video_max_pixels=1024, max_frames=3, out_dtype=dtype)
    one(big, [I.image(2000, 3000), I.clip(3, 2.0, 1500, 2600)])
# a launch large enough for whole-frame items (the row-band instantiation exits at once): 300 two-frame 720p clips
# sharing one frame buffer
wide = vp.VisualPreprocessor(max_frames=2, video_max_pixels=65536, out_dtype=1)
wc = [I.clip(2, 1.0, 720, 1280)] * 300
wpl = wide.plan(wc)
fr = host_frames(O.plan_batch(oracle_params(wide.params), wc[:1])[0])[0]
wbuf, woff, wpit = pack_frames([fr], [3 * 1280])
wide.run(wpl, wbuf, torch.zeros(300, dtype=torch.int64, device="cuda"), wpit.repeat(300), strict=False)
torch.cuda.synchronize()
# the round-2 kernels: u8 HF drop-in resize + linspace sampling, dedup/views, NV12 intake, vision ids, presets
u8 = vp.VisualPreprocessor(max_frames=4, video_max_pixels=20000, image_max_pixels=30000, resize_mode=vp.VP_RESIZE_U8,
                           sampling=vp.VP_SAMPLE_LINSPACE)
one(u8, [I.clip(9, 2.0, 120, 200), I.image(90, 60), I.image(2000, 3000)])
q25 = vp.VisualPreprocessor.from_preset("qwen2_5_vl", max_frames=8, video_max_pixels=50176)
plq = q25.plan([I.clip(300, 29.97, 360, 640), I.clip(50, 10.0, 224, 224)])
q25.second_per_grid(plq)
uc, ul, uid = pre.dedup(mixed, [k // 2 for k in range(len(mixed))])
upl = pre.plan(uc)
pre.views(upl, uid)
H, W, n = 24, 40, 2
nv = torch.randint(0, 256, (n * H * 3 // 2 * W,), dtype=torch.uint8, device="cuda")
rgb = torch.empty(n * H * 3 * W, dtype=torch.uint8, device="cuda")
vp.nv12_to_rgb(nv, nv[H * W:], W, H * 3 // 2 * W, H, W, n, rgb, 3 * W, 3 * W * H)
vp.vision_ids(torch.tensor([[2, 8, 12], [1, 4, 4]], dtype=torch.int64, device="cuda"), 2)
torch.cuda.synchronize()
print("sanitize_run OK")
