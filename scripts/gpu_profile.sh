mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1
python scripts/profile_step.py > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_step.py > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:alt_stage -s 6 -c 1 -o gpurun_out/prof_alt_fwd python scripts/profile_step.py > gpurun_out/ncu_full_fwd.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:alt_stage -s 13 -c 1 -o gpurun_out/prof_alt_inv python scripts/profile_step.py > gpurun_out/ncu_full_inv.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/prof_plain.log; tail -3 gpurun_out/ncu_full_inv.log
