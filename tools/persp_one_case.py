"""One perspective launch of a named tile-class case (for ncu): staged_scale1 / zoomout / border."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_12425_b200 as fv  # noqa: E402
from paper_2505_12425_b200 import synth  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "staged_scale1"
H = {"staged_scale1": [[1.0, 1e-4, 0.3], [-1e-4, 1.0, 0.2], [1e-9, 1e-9, 1.0]],
     "zoomout": [[4.0, 0, 0], [0, 4.0, 0], [1e-9, 1e-9, 1.0]],
     "border": [[1.0, 0, 1e5], [0, 1.0, 0], [0, 0, 1.0]]}[case]
dev = torch.device("cuda", 0)
src = synth.device_u8_batch(16, 2160, 3840, 3, synth.SEED_PERSP, dev)
dst = torch.zeros_like(src)
fv.warp_perspective(src, dst, np.stack([np.array(H)] * 16))
torch.cuda.synchronize()
print("ok", case)
