mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:alt_stage_kernel --launch-skip 7 --launch-count 1 -o gpurun_out/c1 -f python scripts/chain_prof.py > gpurun_out/c1.log 2>&1; echo "chain_prof rc=$?"; tail -2 gpurun_out/c1.log
timeout 600 ncu --set full --clock-control none -k regex:alt_stage_kernel --launch-skip 6 --launch-count 1 -o gpurun_out/c2 -f python scripts/profile_step.py --regen 1 > gpurun_out/c2.log 2>&1; echo "no-import-source rc=$?"; tail -2 gpurun_out/c2.log
timeout 600 ncu --clock-control none -k regex:alt_stage_kernel --launch-skip 6 --launch-count 1 python scripts/profile_step.py --regen 1 > gpurun_out/c3.log 2>&1; echo "basic rc=$?"; tail -2 gpurun_out/c3.log
