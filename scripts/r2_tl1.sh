# 1 GPU: profiled step timelines, this build vs the previous one
for v in prof prof_prev; do
  echo "== $v"
  FC_LIB_PATH=$PWD/_ab/lib_$v.so python scripts/dbg_counters.py 2>&1 | grep -E "pass1:|pass2:|GEMM:|timeline us|first entry|gemm :|anchor" | cut -c1-260
done
