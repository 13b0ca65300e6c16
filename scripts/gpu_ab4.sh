for i in 1 2; do
  for cfg in "ab_old.so" "libfastclip_b200.so"; do
    set -- $cfg
    lib=$1; shift
    env FC_LIB_PATH=$PWD/paper_2407_01445_b200/lib/$lib "$@" timeout -s KILL 200 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>gpurun_out/ab.err
    python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$cfg', round(d['ms_per_step']*1e3,1))" || tail -2 gpurun_out/ab.err
  done
done
