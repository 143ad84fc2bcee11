# C3 (N=4096, tol 1e-10) whole transform on one B200, chunked; oracle on the
# sampled orders only (the every-order parity run is gpu_ooc4096.sh)
mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1
timeout 4000 python scripts/ooc_run.py --n 4096 --tol 1e-10 --chunks 24 --samples 0,1,2048,5000,8191 2> gpurun_out/ooc4096.err > gpurun_out/ooc4096_chain.json; tail -c 1500 gpurun_out/ooc4096_chain.json; tail -3 gpurun_out/ooc4096.err
