mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x -k "real_grid" > gpurun_out/pytest_real.log 2>&1; tail -1 gpurun_out/pytest_real.log
s=$(date +%s); timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$? $(( $(date +%s) - s ))s"
s=$(date +%s); timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$? $(( $(date +%s) - s ))s"
tail -2 gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
