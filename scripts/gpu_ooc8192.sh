mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1
timeout 600 python scripts/ooc_run.py --n 64 --tol 1e-12 --chunks 4 --only 1 --decay 2 --real-grid --samples "" --rows 0,10,63 --out gpurun_out/ooc_small.json 2> gpurun_out/ooc_small.err | tail -c 1500 || { tail -20 gpurun_out/ooc_small.err; exit 1; }
echo
timeout 2400 python scripts/ooc_run.py --n 8192 --tol 1e-10 --chunks 48 --only 0 --decay 2 --real-grid --samples "" --rows 0,5000,8191 2> gpurun_out/ooc8192.err | tail -c 3000; tail -5 gpurun_out/ooc8192.err
