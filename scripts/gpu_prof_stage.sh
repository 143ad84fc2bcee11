mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1
python scripts/stage_times.py --reps 1 > gpurun_out/st_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:alt_stage -s 18 -c 1 -o gpurun_out/prof_v3_fwd6 python scripts/stage_times.py --reps 1 > gpurun_out/ncu_v3.log 2>&1
echo rc=$?; tail -2 gpurun_out/ncu_v3.log
