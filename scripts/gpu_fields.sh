mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -q -m gpu -x -k "fields or pipeline or alt or golden" > gpurun_out/pytest_fields.log 2>&1; tail -3 gpurun_out/pytest_fields.log
timeout 1200 python bench.py --workload c4 --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "c4 rc=$?"; tail -2 gpurun_out/bench_c4.err
cat gpurun_out/bench_c4.json
