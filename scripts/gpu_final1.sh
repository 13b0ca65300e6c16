# 1-GPU evidence: full single-GPU test suite, profiles (bench line, launch list, ncu --set full)
timeout -s KILL 900 python -m pytest tests/ -m gpu -q -x --timeout 600 2>&1 | tail -2
bash scripts/gpu_profiles.sh r1d
