# Profiles for profiles/: environment, ncu launch list of the bench command
# (per-kernel time + DRAM bytes), full captures of the top kernels.
mkdir -p gpurun_out
(free -g; nproc; df -h /dev/shm /tmp; nvidia-smi --query-gpu=name,memory.total --format=csv) > gpurun_out/env.txt 2>&1
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1
timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_plain.json 2> gpurun_out/bench_plain.err; echo "plain rc=$?"
timeout 1500 ncu --target-processes application-only --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
timeout 900 ncu --target-processes application-only --set full --clock-control none --import-source on -k regex:alt_stage -s 6 -c 1 -o gpurun_out/prof_final_fwd python scripts/profile_step.py > gpurun_out/ncu_final.log 2>&1; echo "final rc=$?"

timeout 900 ncu --target-processes application-only --set full --clock-control none --import-source on -k regex:sht_synth -c 1 -o gpurun_out/prof_synth python scripts/profile_step.py > gpurun_out/ncu_synth.log 2>&1; echo "synth rc=$?"
