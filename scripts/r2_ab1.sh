# 1 GPU: the -m gpu suite, then bench lines of this build vs _ab/lib_prev.so (alternating)
timeout -s KILL 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for rep in 1 2 3; do
for v in new prev; do
  unset FC_LIB_PATH; [ $v = prev ] && export FC_LIB_PATH=$PWD/_ab/lib_prev.so
  timeout -s KILL 300 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench N=1 $v', round(d['ms_per_step']*1e3,1), 'us')"
done; done
