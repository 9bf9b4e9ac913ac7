"""Offline shared-memory bank-conflict simulation of K3 (resize_fast_kernel) retired-row layouts at the cfg2
ratio (1280 -> 672, 224-column strips): V retire stores (lane L writes pixels 4L+k) and H tap reads (column
pairs, union start x0(j0+2t) - pa + u), wavefronts per ideal one.  Used to pick vpos()."""
import math
def window(i, inn, out):
    s = inn/out; fs = max(s,1.0); sup = 2*fs; c=(i+0.5)*s
    x0 = max(0, int(c - sup + 0.5)); x1 = min(inn, int(c + sup + 0.5))
    return x0, x1
in_w, out_w = 1280, 672
ws = 224
def layouts():
    yield "natural", lambda x: x
    yield "xor3", lambda x: (x & ~7) | ((x ^ (x >> 3)) & 7)
    yield "subpix", lambda x: (x & ~127) | ((x & 3) << 5) | ((x & 127) >> 2)
    yield "xor2", lambda x: (x & ~7) | ((x ^ (x >> 2)) & 7)
    yield "xor4", lambda x: (x & ~7) | ((x ^ (x >> 4)) & 7)
    yield "xor5", lambda x: (x & ~7) | ((x ^ (x >> 5)) & 7)
    yield "mul3", lambda x: (x & ~7) | ((x*3 + (x>>3)) & 7)
def vstore_cost(f):
    # V lanes L write pixels 4L+k (k=0..3): per instruction k, quarters of 8 lanes
    tot=0
    for w in range(4):
        for k in range(4):
            for q in range(4):
                lanes=[w*128 + 4*(8*q+l) + k for l in range(8)]
                groups={}
                for x in lanes: groups.setdefault(f(x)%8,set()).add(f(x))
                tot+=max(len(v) for v in groups.values())
    return tot/(4*4*4)
def hread_cost(f, strip):
    j0 = strip*ws; jn=min(ws, out_w-j0)
    pa = window(j0, in_w, out_w)[0] & ~15
    npairs = jn//2
    tot=0; n=0
    for u in range(11):
        for wq in range(0, 128, 8):   # quarter-warps of the 128 H lanes
            lanes=[ht for ht in range(wq, wq+8) if ht < npairs]
            if not lanes: continue
            xs=[window(j0+2*ht, in_w, out_w)[0]-pa+u for ht in lanes]
            groups={}
            for x in xs: groups.setdefault(f(x % 512)%8,set()).add(f(x%512))
            tot+=max(len(v) for v in groups.values()); n+=1
    return tot/n
for name,f in layouts():
    print(f"{name:8s} vstore {vstore_cost(f):.2f}  hread " + " ".join(f"{hread_cost(f,s):.2f}" for s in range(3)))
print("---- search")
def subpix_b(B, sh=0):
    # sub-pixel-major within blocks of B pixels (4 sub-pixels), then xor-rotate the 8-granule index by sh
    def f(x):
        base = x & ~(B-1); r = x & (B-1)
        p = ((r & 3) * (B//4)) + (r >> 2)
        return base + p
    return f
def hread_cost_map(f, strip, lmap):
    j0 = strip*ws; jn=min(ws, out_w-j0)
    pa = window(j0, in_w, out_w)[0] & ~15
    npairs = jn//2
    tot=0; n=0
    for u in range(11):
        for w in range(4):
            for q in range(4):
                lanes=[lmap(32*w + 8*q + l) for l in range(8)]
                lanes=[ht for ht in lanes if ht < npairs]
                if not lanes: continue
                xs=[window(j0+2*ht, in_w, out_w)[0]-pa+u for ht in lanes]
                groups={}
                for x in xs: groups.setdefault(f(x % 512)%8,set()).add(f(x%512))
                tot+=max(len(v) for v in groups.values()); n+=1
    return tot/n
lmaps = {"id": lambda t: t,
         "s2": lambda t: (t & ~31) | ((t & 7) * 4 + ((t >> 3) & 3)),   # quarter lanes spaced 4 pairs
         "s4": lambda t: (t & ~31) | (((t & 7) * 4 + ((t >> 3) & 3)) ),
        }
lmaps["odd"] = lambda t: (t & ~31) | (((t & 15) * 2 + ((t >> 4) & 1)))
for B in (16, 32, 64, 128):
    f = subpix_b(B)
    for ln, lm in lmaps.items():
        print(f"subpix{B:<4d} lmap {ln:4s} vstore {vstore_cost(f):.2f} hread " + " ".join(f"{hread_cost_map(f,s,lm):.2f}" for s in range(3)))
for ln, lm in lmaps.items():
    f = lambda x: x
    print(f"natural     lmap {ln:4s} vstore {vstore_cost(f):.2f} hread " + " ".join(f"{hread_cost_map(f,s,lm):.2f}" for s in range(3)))


# ---------------------------------------------------------------------------------------------------------------
# Round 2 (team kernels, whole-row or sliced footprints): retired-row layouts x H tap order.  H lane q owns column
# pair (2q, 2q+1); its UL-tap union window starts at x0(2q).  "rotation" = the tap order of lane q: at instruction t
# it reads position x0 + ((t + r_q) mod UL).  Wavefronts per quarter-warp (8 lanes x 16 B), 1.0 = conflict-free.
# Result: layout rpos(x) = (x & ~7) | ((x + 5 (x >> 3)) & 7) with r_q = -x0 mod UL (every lane
# reads one residue class mod UL per instruction) is conflict-free for V stores and H reads at every ratio below.
def team_cost(inn, out, layout, rot, UL=10):
    Q = out // 2
    st = [window(2 * q, inn, out)[0] for q in range(Q)]
    tot = n = 0
    for t in range(UL):
        for l0 in range(0, Q, 8):
            g = [layout(st[q] + ((t + rot(q % 32, st[q])) % UL)) for q in range(l0, min(l0 + 8, Q))]
            cls = {}
            for x in g:
                cls.setdefault(x % 8, set()).add(x)
            tot += max(len(v) for v in cls.values())
            n += 1
    return tot / n


def team_vstore_cost(layout):
    tot = n = 0
    for j in range(4):
        for l0 in range(0, 320, 8):
            g = [layout(4 * L + j) for L in range(l0, l0 + 8)]
            cls = {}
            for x in g:
                cls.setdefault(x % 8, set()).add(x)
            tot += max(len(v) for v in cls.values())
            n += 1
    return tot / n


if __name__ == "__main__":
    tpos = lambda x: (x & ~31) | ((x & 3) << 3) | ((x & 31) >> 2)
    rpos = lambda x: (x & ~7) | ((x + 5 * (x >> 3)) & 7)
    ratios = [(1280, 672), (720, 384), (854, 672), (640, 336), (1000, 640), (1920, 1088), (1280, 1024)]
    for name, lay, rot in (("round-1 sub-pixel-major, no rotation", tpos, lambda q, x: 0),
                           ("rpos, rotation -x0 mod UL", rpos, lambda q, x: -x)):
        print(f"{name:40s} V stores {team_vstore_cost(lay):.2f}  H reads",
              [round(team_cost(i, o, lay, rot), 3) for i, o in ratios])
