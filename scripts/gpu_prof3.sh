mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1
python scripts/stage_times.py --reps 1 > gpurun_out/st_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:alt_stage -s 2 -c 1 -o gpurun_out/prof_bf0 python scripts/stage_times.py --reps 1 > gpurun_out/ncu_bf0.log 2>&1 && \
python scripts/profile_step.py > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sht_synth -c 1 -o gpurun_out/prof_synth python scripts/profile_step.py > gpurun_out/ncu_synth.log 2>&1
echo rc=$?
