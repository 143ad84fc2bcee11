mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1
python scripts/profile_step.py --n 512 --regen 1 > gpurun_out/ps.log 2>&1; cat gpurun_out/ps.log
S=$(grep "stages fwd/inv" gpurun_out/ps.log | awk '{print $3}')
timeout 900 ncu --target-processes application-only --set full --clock-control none --import-source on -k regex:alt_stage -s $((S-1)) -c 1 -o gpurun_out/prof_regen1 python scripts/profile_step.py --n 512 --regen 1 > gpurun_out/ncu_regen.log 2>&1
echo rc=$?; tail -2 gpurun_out/ncu_regen.log
timeout 900 ncu --target-processes application-only --set full --clock-control none --import-source on -k regex:alt_stage -s $((S-1)) -c 1 -o gpurun_out/prof_regen0 python scripts/profile_step.py --n 512 --regen 0 > gpurun_out/ncu_regen0.log 2>&1 || true
echo rc=$?
