# r1h: config 3 at full table size (N = 315M) parity on one B200
mkdir -p gpurun_out/r1h
timeout -s KILL 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q --timeout 600 -k "315000000" > gpurun_out/r1h/pytest_315m.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r1h/pytest_315m.log
free -g | head -2
