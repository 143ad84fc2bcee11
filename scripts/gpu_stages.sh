mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1
python scripts/stage_times.py > gpurun_out/stages.jsonl 2> gpurun_out/stages.err; echo rc=$?
cat gpurun_out/stages.jsonl; tail -3 gpurun_out/stages.err
