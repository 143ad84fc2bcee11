mkdir -p gpurun_out
nproc; free -g | head -2; df -h /dev/shm /tmp | tail -2
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_ooc.py -x -q > gpurun_out/pytest_ooc.log 2>&1; tail -15 gpurun_out/pytest_ooc.log
timeout 900 python scripts/ooc_run.py --n 1024 --tol 1e-12 --chunks 4 --samples 1,500,1500,2047 --rows 0,300,1023 2> gpurun_out/ooc1024.err | tail -c 2500; tail -5 gpurun_out/ooc1024.err
