set -x
mkdir -p gpurun_out
timeout -s KILL 400 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "bench rc=$?"
tail -3 gpurun_out/bench1.err; cat gpurun_out/bench1.json
for s in 1 2 4 8; do FC_GEMM_SPLIT=$s timeout -s KILL 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('split',$s, d['ms_per_step'], d['phases_ms'])"; done
