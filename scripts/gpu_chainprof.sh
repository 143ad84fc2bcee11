mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1
timeout 600 python scripts/stage_times.py --reps 5 > gpurun_out/stage_times.jsonl 2> gpurun_out/stage_times.err; echo "st rc=$?"
timeout 900 ncu --target-processes application-only --set full --clock-control none --import-source on -k regex:alt_stage -s 2 -c 1 -o gpurun_out/prof_chain2 python scripts/stage_times.py --reps 1 > gpurun_out/ncu_chain2.log 2>&1; echo "ncu rc=$?"
