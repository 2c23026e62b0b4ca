"""One four-step NDCT and NDCT^T at 2^log2n, world 1 (for ncu launch lists)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1505_00354_b200 as fl  # noqa: E402
from paper_1505_00354_b200 import distributed as D  # noqa: E402

log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 26
n = 1 << log2n
cfg = fl.TransformConfig(n)
c = torch.from_numpy(fl.random_decaying(n, 1.0, 3)).cuda()
fs = D.FourStep(cfg, 1, 0)
comm = D.TorchComm(None)
chat = fs.to_residue(c)
g = fs.groups()
for _ in range(2):
    D._ndct_four_step(fs, comm, chat, g)
    D._ndct_t_four_step(fs, comm, c, g)
torch.cuda.synchronize()
print("ok", g)
