# 1 GPU: profiled timeline of this build, then bench lines of this build vs _ab/lib_prev.so (alternating)
FC_LIB_PATH=$PWD/_ab/lib_prof.so python scripts/dbg_counters.py 2>&1 | grep -E "pass1:|pass2:|GEMM:|first entry|gemm :|anchor" | cut -c1-250
for rep in 1 2 3; do
for v in new prev; do
  unset FC_LIB_PATH; [ $v = prev ] && export FC_LIB_PATH=$PWD/_ab/lib_prev.so
  python bench.py --steps 50 --warmup 5 --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench N=1 $v', round(d['ms_per_step']*1e3,1), 'us')"
done; done
