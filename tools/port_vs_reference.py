"""One-core wall time of the unmodified reference `_resize_u8` (app.py:64-78, imported
from /root/reference, build container only) against the oracle port bench.py times,
on the same frame, with an equality check. Not run on the GPU box."""
import sys, time, numpy as np
sys.path.insert(0, '/root/reference/pkg/src'); sys.path.insert(0, '/root/repo')
from fovea.service.app import _resize_u8
from fovea.image import Image, ImageSize
from fovea.tensor import Tensor
from oracle import fovea_oracle as O
a = O.seeded_u8_image(3840, 2160, 3, 1)
img = Image(Tensor.from_shape_slice(a.shape, a.reshape(-1), dtype=np.uint8), 3) if hasattr(Tensor,'from_shape_slice') else None
def t(f, n=3):
    f(); ts=[]
    for _ in range(n):
        s=time.perf_counter(); r=f(); ts.append(time.perf_counter()-s)
    return min(ts), r
tr, r = t(lambda: _resize_u8(img, ImageSize(1920,1080), 'bilinear'))
to, o = t(lambda: O.resize_u8(a, 1920, 1080))
print('down  ref %.3fs port %.3fs  equal %s' % (tr, to, np.array_equal(r.as_array().reshape(o.shape), o)))
a2 = a[:540, :960].copy()
img2 = Image(Tensor.from_shape_slice(a2.shape, a2.reshape(-1), dtype=np.uint8), 3)
tr, r = t(lambda: _resize_u8(img2, ImageSize(1920,1080), 'bilinear'))
to, o = t(lambda: O.resize_u8(a2, 1920, 1080))
print('up2   ref %.3fs port %.3fs  equal %s' % (tr, to, np.array_equal(r.as_array().reshape(o.shape), o)))
from fovea import imgproc
g = O.seeded_u8_image(1920, 1080, 3, 2)
gsrc = Image(Tensor.from_shape_slice(g.shape, g.reshape(-1), dtype=np.uint8), 3)
gdst = Image(Tensor.from_shape_slice((1080, 1920, 1), np.zeros(1080 * 1920, np.uint8), dtype=np.uint8), 1)
tr, _ = t(lambda: imgproc.gray_from_rgb(gsrc, gdst))
to, o = t(lambda: O.gray_from_rgb(g))
print('gray  ref %.3fs port %.3fs  equal %s' % (tr, to, np.array_equal(gdst.as_array().reshape(o.shape), o)))
