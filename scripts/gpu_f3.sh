# f3: device entry tabulation — planning wall time host vs device
mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
export BFSHT_PLAN_TRACE=1
timeout 300 python scripts/plan_times.py --n 4096 --orders 16 --processes 4 > gpurun_out/plan_small.json 2> gpurun_out/plan_small.err; echo rc=$?; tail -3 gpurun_out/plan_small.json; tail -25 gpurun_out/plan_small.err
