"""Run one K5 v2 (TMA stencil) launch of the given H W pitch in mode none (dev tool, e.g. under compute-sanitizer).
  python tools/stencil_tma_small.py H W pitch
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
from paper_2401_09290_b200 import devmem, guardian as g
MiB=1<<20
a=g.Arena(0, 32*MiB); p=a.partition_alloc(16*MiB)
devmem.view(p.base+MiB, 1<<16, torch.float32).uniform_(0,1)
H,W,pitch=int(sys.argv[1]),int(sys.argv[2]),int(sys.argv[3])
a.stencil_tma(p.id, "none", p.base+8*MiB, p.base+MiB, H, W, pitch, 0.5, 0.125)
torch.cuda.synchronize()
print("ok", H, W, pitch)
