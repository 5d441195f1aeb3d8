import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_2505_12425_b200 as fv
from paper_2505_12425_b200 import synth, _native, _tensors
dev = torch.device("cuda", 0)
src = synth.device_u8_batch(64, 2160, 3840, 3, 1, dev)
down = torch.zeros((64, 1080, 1920, 3), dtype=torch.uint8, device=dev)
small_s = torch.zeros((2, 64, 64, 3), dtype=torch.uint8, device=dev)
small_d = torch.zeros((2, 32, 32, 3), dtype=torch.uint8, device=dev)
for _ in range(3): fv.resize_bilinear_u8(small_s, small_d)
torch.cuda.synchronize()
t=time.perf_counter()
for _ in range(100): fv.resize_bilinear_u8(small_s, small_d)
t1=time.perf_counter(); torch.cuda.synchronize(); t2=time.perf_counter()
print("python call (small) %.1f us/call, drain %.1f us" % ((t1-t)/100*1e6, (t2-t1)*1e6))
# pieces
t=time.perf_counter()
for _ in range(1000): s=_tensors.as_image(small_s,"src"); d=_tensors.as_image(small_d,"dst")
print("as_image x2 %.1f us" % ((time.perf_counter()-t)/1000*1e6))
t=time.perf_counter()
for _ in range(1000): _tensors.check_distinct(small_s, small_d)
print("check_distinct %.1f us" % ((time.perf_counter()-t)/1000*1e6))
t=time.perf_counter()
for _ in range(1000): _tensors.stream_ptr(small_s)
print("stream_ptr %.1f us" % ((time.perf_counter()-t)/1000*1e6))
t=time.perf_counter()
for _ in range(1000):
    with torch.cuda.device(dev): pass
print("device ctx %.1f us" % ((time.perf_counter()-t)/1000*1e6))
s=_tensors.as_image(small_s,"src"); d=_tensors.as_image(small_d,"dst"); sp=_tensors.stream_ptr(small_s)
t=time.perf_counter()
for _ in range(1000):
    _native.call("fv_resize_bilinear_u8", s.ptr, s.img_stride, s.row_pitch, s.h, s.w, d.ptr, d.img_stride, d.row_pitch, d.h, d.w, s.c, s.n, sp)
t1=time.perf_counter(); torch.cuda.synchronize()
print("raw ctypes call+launch %.1f us" % ((t1-t)/1000*1e6))
# big kernel: host time per call when queue is busy
torch.cuda.synchronize()
t=time.perf_counter()
for _ in range(5): fv.resize_bilinear_u8(src, down)
t1=time.perf_counter(); torch.cuda.synchronize(); t2=time.perf_counter()
print("big: host %.1f us/call, total %.3f ms/call" % ((t1-t)/5*1e6, (t2-t)/5*1e3))
