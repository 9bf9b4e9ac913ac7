"""Debug: which pixels of the smoke batch disagree, per sub-batch combination."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import oracle as O, vp_inputs as I, paper_2604_16893_b200 as vp
from parity import pixel_failures

params, c1 = I.config("cfg1")
combos = {"all": c1 + [I.image(100, 60), I.clip(9, 2.0, 70, 100)], "img": [I.image(100, 60)],
          "img+team": [I.image(100, 60), I.clip(9, 2.0, 70, 100)], "copy+img": c1 + [I.image(100, 60)],
          "team+img": [I.clip(9, 2.0, 70, 100), I.image(100, 60)], "team": [I.clip(9, 2.0, 70, 100)]}
for name, clips in combos.items():
    pre = vp.VisualPreprocessor(device="cuda:0", **params)
    pl = pre.plan(clips)
    oplans, _ = O.plan_batch(dict(params), clips)
    frames = [I.frames_u8("noise", k, o.idx, o.in_h, o.in_w) for k, o in enumerate(oplans)]
    off, pitch, total = pre.frames_layout(pl)
    buf = np.zeros(total, np.uint8)
    for k, fr in enumerate(frames):
        v = buf[off[k]: off[k] + fr.shape[0] * fr.shape[1] * pitch[k]].reshape(fr.shape[0], fr.shape[1], pitch[k])
        v[:, :, :3 * fr.shape[2]] = fr.reshape(fr.shape[0], fr.shape[1], -1)
    out = pre.run(pl, torch.from_numpy(buf).cuda(), torch.from_numpy(off).cuda(), torch.from_numpy(pitch).cuda())
    ref = O.process_batch(dict(params), clips, frames, plans=oplans)
    print(name, "variants", pl.plans_host["kernel_variant"][:len(clips)].tolist(), "pitch", pitch.tolist())
    for key, rk in (("pixel_values", "pixel_values_images"), ("pixel_values_videos", "pixel_values_videos")):
        g = out[key].cpu()
        if g.numel() == 0:
            continue
        bad = pixel_failures(g, ref[rk])
        if bad.any():
            rows = np.unique(np.argwhere(bad)[:, 0])
            print("  ", key, int(bad.sum()), "bad of", bad.size, "rows", rows[:10], "...", len(rows))
        else:
            print("  ", key, "ok")
