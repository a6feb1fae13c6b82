"""Layout study (DESIGN.md (d)): distinct 32-B sectors and 128-B lines one
warp's gather touches per voxel-step, linear x-fastest vs bricked layouts, on
the walk's own access pattern -- 8x4 ray quads of the C2 geometry stepping in
lock-step (each ray's k-th segment voxel from the reference's
python_ref.ray_structure, oracle/_ref).  Measurement script, CPU only.
Result at C2 (6 narrow poses x 6 quads): linear 20.2 sectors / 19.2 lines per
request (ncu: 19.4 sectors), 4x4x4 bricks 18.4 / 12.1, 8x4x2 20.2 / 12.8,
2x2x2 18.6 / 12.5.
"""
import os
import sys, math, numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, 'oracle', '_ref')); sys.path.insert(0, ROOT)
import drrtrace as dt
from drrtrace._kernels import python_ref
from paper_2208_12737_b200 import synthetic
dims=(512,512,133); sp=(0.703125,0.703125,2.5)
vol=dt.Volume(dims, sp, (0,0,0), np.zeros(dims))
spec=dt.DetectorSpec.for_volume(vol,200,200,(3.6,3.6))
from drrtrace.geometry import detector_grid
def addr_linear(f):
    return 4*f
def make_brick(bx,by,bz):
    nbx=-(-dims[0]//bx); nby=-(-dims[1]//by)
    def a(f):
        i=f%dims[0]; j=(f//dims[0])%dims[1]; k=f//(dims[0]*dims[1])
        b=(i//bx)+nbx*((j//by)+nby*(k//bz))
        return 4*(b*bx*by*bz+(i%bx)+bx*((j%by)+by*(k%bz)))
    return a
layouts={'linear':addr_linear,'b4x4x4':make_brick(4,4,4),'b8x4x2':make_brick(8,4,2),'b4x4x2':make_brick(4,4,2),'b8x8x1':make_brick(8,8,1),'b2x2x2':make_brick(2,2,2)}
rng=np.random.default_rng(0)
poses=synthetic.sample_poses((300,math.pi/2,math.pi/2,0,0,0,0), synthetic.NARROW_HALF_WIDTHS, 6, seed=0)
res={k:[0,0,0] for k in layouts}
for eta in poses:
    rays=detector_grid(dt.PoseParameters.from_vector(eta), spec)
    pix=rays.pixels.reshape(200,200,3)
    for trial in range(6):
        h0=rng.integers(0,196); w0=rng.integers(0,192)
        quad=pix[h0:h0+4, w0:w0+8].reshape(-1,3)   # 8 wide x 4 high warp quad
        labels,use,flat,miss=python_ref.ray_structure(None,dims,sp,(0,0,0),rays.source,quad)
        T=flat.shape[1]
        for t in range(T):
            f=flat[:,t]; u=use[:,t]
            fs=f[u & (f>=0)]
            if len(fs)==0: continue
            for k,fn in layouts.items():
                ad=np.array([fn(int(x)) for x in fs])
                res[k][0]+=len(set(ad//32)); res[k][1]+=len(set(ad//128)); res[k][2]+=1
for k,(s,l,n) in res.items(): print(f"{k:8s} sectors/req {s/n:6.2f}  lines/req {l/n:6.2f}")
