mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
CACHE=/tmp/ec timeout 900 python scripts/e2e_steps.py 2>&1 | tail -10
