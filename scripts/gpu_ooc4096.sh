# C3 (N=4096, tol 1e-10) whole transform on one B200, chunked, with the
# oracle run on every order (--oracle-all: global parity vs pocketfft oracle)
mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1
( while true; do free -g | sed -n 2p; nvidia-smi --query-gpu=memory.used --format=csv,noheader; sleep 60; done ) > gpurun_out/ooc4096_mem.log 2>&1 &
timeout 5400 python scripts/ooc_run.py --n 4096 --tol 1e-10 --chunks 24 --samples 0,1,2048,5000,8191 --oracle-all 2> gpurun_out/ooc4096.err | tail -c 3000; tail -5 gpurun_out/ooc4096.err
