mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1
timeout 600 python scripts/fields_step.py
# stage launches of one fields pass: fields_pack, 7 forward stages, assemble; the 7th stage (index 6) is the final one
timeout 900 ncu --target-processes application-only --set full --clock-control none --import-source on -k regex:alt_stage -s 6 -c 1 -o gpurun_out/prof_fields_final python scripts/fields_step.py > gpurun_out/ncu_ff.log 2>&1; echo "rc=$?"
