import sys, numpy as np, torch
sys.path.insert(0,'.')
import paper_2505_12425_b200 as fv, oracle as O
rng=np.random.default_rng(1)
h,w,c=75,96,3
for dt in (np.uint8, np.float32):
    a=rng.integers(0,256,(h,w,c),dtype=np.uint8)
    if dt==np.float32: a=(a/np.float32(255)).astype(np.float32)
    invs=[np.array([[0.0,1.0,0.0],[-1.0,0.0,h-1.0]]),np.array([[0.0,-1.25,80.0],[1.25,0.0,-7.0]]),np.array([[1.0,0.0,0.5],[0.0,1.0,-0.5]]),
          np.array([[1.0,0.0,32.0],[0.0,1.0,24.0]]),np.array([[-1.0,0.0,w-1.0],[0.0,1.0,0.0]]),np.array([[0.5,0.0,-10.0],[0.0,0.5,40.0]]),np.array([[1.0,1e-17,3.0],[0.0,1.0,2.0]])]
    for k,inv in enumerate(invs):
        for oh,ow,b in [(h,w,0),(100,130,5)]:
            bb=b if dt==np.uint8 else b/255.0
            dst=torch.zeros((oh,ow,c),dtype=torch.from_numpy(a).dtype,device='cuda')
            fv.warp_affine(torch.from_numpy(a).cuda(),dst,inv,border=bb,inverse=True)
            got=dst.cpu().numpy(); ref=O.warp_affine(a,inv,oh,ow,border=bb)
            bad=np.argwhere((got!=ref).any(-1))
            print(dt.__name__,k,oh,ow,b,'bad',len(bad), bad[:5].tolist(), [ (got[tuple(p)].tolist(), ref[tuple(p)].tolist()) for p in bad[:3]])
