import os, sys
sys.path.insert(0, "tests"); sys.path.insert(0, "oracle"); sys.path.insert(0, ".")
from gpu_helpers import run_pair, norm_rel
B, d = int(sys.argv[1]), int(sys.argv[2])
res, _, _, _ = run_pair("fastclip_v3", B=B, d=d, N=5000, steps=1, seed=5)
got, ref = res[0]
print(B, d, os.environ.get("FC_SHARED_Q"), "dE1", norm_rel(got["dE1"], ref["dE1"]), "dE2", norm_rel(got["dE2"], ref["dE2"]), flush=True)
