# compute-sanitizer over a small step sequence (one tool per call: TOOL=memcheck|racecheck|synccheck)
mkdir -p gpurun_out/r2e
cat > /tmp/san_step.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests")); sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
os.environ.setdefault("FC_GRAPH", "0")
from gpu_helpers import run_pair, norm_rel
for v in ("fastclip_v3", "fastclip_v2"):
    res, _, _, _ = run_pair(v, B=256, d=128, N=2048, steps=2, seed=3)
    print(v, "dE1 err", max(norm_rel(g["dE1"], r["dE1"]) for g, r in res))
PY
timeout -s KILL 1500 compute-sanitizer --tool ${TOOL} --target-processes all --print-limit 20 python /tmp/san_step.py > gpurun_out/r2e/sanitizer_${TOOL}.log 2>&1; echo "rc=$?"
tail -15 gpurun_out/r2e/sanitizer_${TOOL}.log
