# Final evidence pass: bench line, ncu launch list of the same command,
# --set full captures of the final ALT stage and the DFT synthesis.
mkdir -p gpurun_out
(free -g; nproc; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv) > gpurun_out/env.txt 2>&1
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_v9.json 2> gpurun_out/bench_v9.err; echo "bench rc=$?"
timeout 1500 ncu --target-processes application-only --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_bench_v9.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
timeout 900 ncu --target-processes application-only --set full --clock-control none --import-source on -k regex:alt_stage -s 6 -c 1 -o gpurun_out/prof_final_fwd_v9 python scripts/profile_step.py > gpurun_out/ncu_final.log 2>&1; echo "final rc=$?"
timeout 900 ncu --target-processes application-only --set full --clock-control none --import-source on -k regex:sht_synth -c 1 -o gpurun_out/prof_synth_v9 python scripts/profile_step.py > gpurun_out/ncu_synth.log 2>&1; echo "synth rc=$?"
