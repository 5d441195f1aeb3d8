import numpy as np, sys
sys.path.insert(0, '.')
from paper_2505_12425_b200 import io as fio
z = np.load('tests/golden/jpeg.npz')
names = sorted({k.split('__')[0] for k in z.files if k.endswith('__out')})
for n in names:
    h0 = fio.stats["host_entropy"]
    fio.decode_jpeg_batch([z[n + '__jpg'].tobytes()], entropy='gpu')
    if fio.stats["host_entropy"] != h0: print("fallback:", n)
