# f3: planning wall time, host vs device entry tabulation, N=4096
mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout 1500 python scripts/plan_times.py --n 4096 --orders 512 > gpurun_out/plan_times_n4096_512.json 2> gpurun_out/plan_times_512.err; echo rc=$?; cat gpurun_out/plan_times_n4096_512.json; tail -3 gpurun_out/plan_times_512.err
