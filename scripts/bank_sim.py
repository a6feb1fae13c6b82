"""Plane-table bank-conflict study: shared-memory
wavefronts per warp voxel-step of the walk's plane-table LDS.64 under
candidate table layouts, on the walk's own access pattern -- 8x4 ray quads of
the C2 geometry stepping in lock-step over the chest phantom, each ray walked
over its nonzero span (the trimmed walk's approximate extent).  Each lane
reads the next plane of the axis it just crossed.  Bank model: 64-bit loads
are served per half-warp, one wavefront per distinct 8-byte word in the most
loaded of 16 eight-byte bank slots.  Measurement script, CPU only.
Result at C2 (4 narrow poses x 6 quads; ncu: 3.7 wavefronts per warp step):
current concatenated tables 3.74, per-axis padding 3.72, axes interleaved with
stride 4 4.51, slot groups (dominant axis 8 even slots, others 4 + 4) 3.67,
plus warp-aligned starts 3.59; 4-wide x 8-high quads (`--quad 4x8`, current
tables) 3.41.
"""
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2208_12737_b200 import synthetic  # noqa: E402
import torch  # noqa: E402
from paper_2208_12737_b200.geometry import pose_frames  # noqa: E402

dims = (512, 512, 133)
sp = (0.703125, 0.703125, 2.5)
org = (0.0, 0.0, 0.0)
PAD = 3
vol = synthetic.chest_phantom(dims)


def walk_reads(src, pix, align_D=None):
    """Per ray: the list of (axis, plane index) the lean walk reads, over the
    ray's nonzero span."""
    d = pix - src
    out = []
    for r in range(pix.shape[0]):
        dv = d[r]
        cands = []
        for a in range(3):
            if dv[a] == 0:
                continue
            k = np.arange(dims[a] + 1)
            al = (org[a] + k * sp[a] - src[a]) / dv[a]
            cands.append(np.stack([al, np.full(k.shape, a), k], 1))
        c = np.concatenate(cands)
        lo = max(0.0, max(min((org[a] - src[a]) / dv[a], (org[a] + dims[a] * sp[a] - src[a]) / dv[a])
                              for a in range(3) if dv[a] != 0))
        hi = min(1.0, min(max((org[a] - src[a]) / dv[a], (org[a] + dims[a] * sp[a] - src[a]) / dv[a])
                          for a in range(3) if dv[a] != 0))
        if not lo < hi:
            out.append([])
            continue
        c = c[(c[:, 0] >= lo) & (c[:, 0] <= hi)]
        c = c[np.argsort(c[:, 0], kind="stable")]
        al = np.concatenate([[lo], c[:, 0], [hi]])
        mid = 0.5 * (al[:-1] + al[1:])
        pos = src[None, :] + mid[:, None] * dv[None, :]
        idx = np.clip(np.floor((pos - np.array(org)) / np.array(sp)), 0, np.array(dims) - 1).astype(int)
        val = vol[idx[:, 0], idx[:, 1], idx[:, 2]]
        nz = np.nonzero(val)[0]
        if len(nz) == 0:
            out.append([])
            continue
        st = np.sign(dv).astype(int)
        out.append((c, nz[0], nz[-1], st))
    if align_D is None:
        return [[(int(a), int(k) + st[int(a)]) for _, a, k in c[b:e]] if len(x) else []
                for x in out for (c, b, e, st) in [x if len(x) else (None, 0, 0, None)]]
    # warp-aligned starts: every lane starts at the warp's earliest start plane
    # on the dominant axis (in the walking direction)
    D = align_D
    starts = []
    for x in out:
        if not len(x):
            continue
        c, b, e, st = x
        dm = c[:b + 1][c[:b + 1, 1] == D]
        starts.append(int(dm[-1, 2]) * st[D] if len(dm) else -10**9)
    k0 = min(starts) if starts else 0
    res = []
    for x in out:
        if not len(x):
            res.append([])
            continue
        c, b, e, st = x
        m = np.nonzero((c[:, 1] == D) & (c[:, 2] * st[D] >= k0))[0]
        b2 = min(b, int(m[0])) if len(m) else b
        res.append([(int(a), int(k) + st[int(a)]) for _, a, k in c[b2:e]])
    return res


def layouts(D):
    n = [dims[0] + 1 + 2 * PAD, dims[1] + 1 + 2 * PAD, dims[2] + 1 + 2 * PAD]
    base = [PAD, n[0] + PAD, n[0] + n[1] + PAD]
    A, B = [a for a in range(3) if a != D]
    part = {D: (2, 0), A: (4, 1), B: (4, 3)}
    def part8(e):  # axis e gets the 8 even slots, the others 4 each
        o1, o2 = [a for a in range(3) if a != e]
        m = {e: (2, 0), o1: (4, 1), o2: (4, 3)}
        return lambda a, k: m[a][0] * (k + PAD) + m[a][1]
    return {
        "part8_x": part8(0), "part8_y": part8(1), "part8_z": part8(2),
        "concat": lambda a, k: base[a] + k,
        "inter4": lambda a, k: 4 * (k + PAD) + a,
        "part_D2": lambda a, k: part[a][0] * (k + PAD) + part[a][1],
        "concat_pad8": lambda a, k: base[a] + 8 * a + k,
    }


def wavefronts(reads_by_lane, fn):
    T = max(len(x) for x in reads_by_lane)
    tot = steps = 0
    for t in range(T):
        w = 0
        active = False
        for half in (range(0, 16), range(16, 32)):
            words = {fn(*reads_by_lane[l][t]) for l in half if t < len(reads_by_lane[l])}
            if not words:
                continue
            active = True
            slots = np.bincount(np.array([x % 16 for x in words]), minlength=16)
            w += int(slots.max())
        if active:
            tot += w
            steps += 1
    return tot, steps


def main(n_poses=4, quads=6, qw=8):
    rng = np.random.default_rng(0)
    poses = synthetic.sample_poses((300, math.pi / 2, math.pi / 2, 0, 0, 0, 0),
                                   synthetic.NARROW_HALF_WIDTHS, n_poses, seed=0)
    center = tuple(0.5 * dims[a] * sp[a] for a in range(3))
    res = {}
    for eta in poses:
        f = pose_frames(torch.tensor(np.asarray(eta, float)[None]), center)[0].numpy()
        src, p0, eh, ew = f[0:3], f[3:6], 3.6 * f[6:9], 3.6 * f[9:12]
        dD = np.abs(p0 - src) / np.array(sp)
        D = int(np.argmax(dD))
        for _ in range(quads):
            h0, w0 = rng.integers(40, 156), rng.integers(40, 150)
            lanes = []
            for lane in range(32):
                h, w = h0 + lane // qw, w0 + lane % qw
                lanes.append(p0 + (h - 99.5) * eh + (w - 99.5) * ew)
            for tag, al in (("", None), ("+align", D)):
                reads = walk_reads(src, np.array(lanes), al)
                for name, fn in layouts(D).items():
                    t, s = wavefronts(reads, fn)
                    a = res.setdefault(name + tag, [0, 0, 0])
                    a[0] += t
                    a[1] += s
                    a[2] += sum(len(x) for x in reads)
    for name, (t, s, n) in res.items():
        print(f"{name:18s} wavefronts per warp step {t / s:5.2f}  warp steps {s}  "
              f"lane steps {n}  wavefronts {t}")


if __name__ == "__main__":
    qw = 8
    if "--quad" in sys.argv:
        qw = int(sys.argv[sys.argv.index("--quad") + 1].split("x")[0])
    main(qw=qw)
