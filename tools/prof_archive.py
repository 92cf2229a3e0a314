"""One exact-mode archive compress of a 256^3 x 32 device field (ncu target)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_01380_b200 import archive as A  # noqa: E402

mode = A.ARCHIVE_SKETCH if "--sketch" in sys.argv else A.ARCHIVE_EXACT
g, n = 256, 32
field = torch.randn((n, g ** 3), dtype=torch.float64, device="cuda").T
kw = dict(mode=mode, ell=16, seed=1) if mode == A.ARCHIVE_SKETCH else {}
data = A.compress_field(field, (g,) * 3, (4,) * 3, (2,) * 3, periodic=(1, 1, 1), rank=8, **kw)
torch.cuda.synchronize()
print("archive bytes", len(data))
