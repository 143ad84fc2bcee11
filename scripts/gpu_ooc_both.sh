mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1
timeout 1500 python scripts/ooc_run.py --n 8192 --tol 1e-10 --chunks 48 --only 0 --decay 2 --real-grid --samples "" --rows 0,5000,8191 2> gpurun_out/ooc8192.err | tail -c 600; tail -3 gpurun_out/ooc8192.err
timeout 3000 python scripts/ooc_run.py --n 4096 --tol 1e-10 --chunks 24 2> gpurun_out/ooc4096.err | tail -c 600; tail -3 gpurun_out/ooc4096.err
