# r02 evidence: round-end sequence (smoke, pytest -m gpu, default bench), the
# ncu launch list of the bench command (plans from the packed cache so no
# process pool runs under ncu), and the reference-arm line
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"; tail -c 400 gpurun_out/bench_default.json
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --plan-cache /tmp/pc > gpurun_out/bench_cachewrite.json 2>&1; echo "cache rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_launches_bench_n1024.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --plan-cache /tmp/pc > gpurun_out/ncu_bench.log 2>&1; echo "ncu rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; tail -c 300 gpurun_out/bench_ref.json
