mkdir -p gpurun_out
timeout -s KILL 200 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_plain.json 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
echo done
