"""Runs a few FastCLIP steps at a given shape (for ncu captures): warmup + measured steps."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_01445_b200 as P  # noqa: E402
from paper_2407_01445_b200 import synthetic as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=5120)
ap.add_argument("--dim", type=int, default=512)
ap.add_argument("--n-train", type=int, default=2_700_000)
ap.add_argument("--variant", default="fastclip_v3")
ap.add_argument("--steps", type=int, default=3)
a = ap.parse_args()
B, d = a.batch, a.dim
cfg = P.config_defaults(a.variant, a.n_train, dim=d, local_batch=B)
step = P.LossStep(cfg)
step.load_tables(u1=S.warm_u(a.n_train, 1), u2=S.warm_u(a.n_train, 2))
b1, b2 = S.embeddings(B, d, 0)
e1 = torch.from_numpy(b1.view(np.int16)).cuda().view(torch.bfloat16)
e2 = torch.from_numpy(b2.view(np.int16)).cuda().view(torch.bfloat16)
ids = torch.from_numpy(S.ids(B, a.n_train, 0)).cuda()
for _ in range(a.steps):
    step.step(e1, e2, ids, 0.6, 1e-14)
torch.cuda.synchronize()
print("ok", step.scalars())
