# whole SHT at N=2048 on one GPU (L = 8191 prime: Bluestein phi rows), with the oracle check
mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; exit 1; }
( while true; do free -g | sed -n 2p; nvidia-smi --query-gpu=memory.used --format=csv,noheader; sleep 60; done ) > gpurun_out/n2048_mem.log 2>&1 &
timeout 2400 python bench.py --n 2048 --steps 10 --warmup 3 > gpurun_out/bench_n2048.json 2> gpurun_out/bench_n2048.err; echo rc=$?
tail -c 1500 gpurun_out/bench_n2048.json; tail -3 gpurun_out/bench_n2048.err
