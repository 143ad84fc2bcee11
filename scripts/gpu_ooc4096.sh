mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_ooc.py -x -q > gpurun_out/pytest_ooc.log 2>&1; tail -2 gpurun_out/pytest_ooc.log
( while true; do free -g | sed -n 2p; nvidia-smi --query-gpu=memory.used --format=csv,noheader; sleep 60; done ) > gpurun_out/ooc4096_mem.log 2>&1 &
timeout 4200 python scripts/ooc_run.py --n 4096 --tol 1e-10 --chunks 24 2> gpurun_out/ooc4096.err | tail -c 3000; tail -5 gpurun_out/ooc4096.err
