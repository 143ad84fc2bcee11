# session check: smoke + pytest -m gpu + default bench + per-stage ALT times
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"; tail -c 600 gpurun_out/bench_default.json
timeout 600 python scripts/stage_times.py --n 1024 > gpurun_out/stage_times_n1024.jsonl 2>&1; tail -30 gpurun_out/stage_times_n1024.jsonl
