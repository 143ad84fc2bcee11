# r02 evidence: round-end sequence (smoke, pytest -m gpu, default bench), the
# ncu launch list of the bench command (plans from the packed cache so no
# process pool runs under ncu), a --set full capture of the forward chain
# stages (alt_chain_kernel) and of the final forward stage, per-stage times,
# and the reference-arm line
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"; tail -c 400 gpurun_out/bench_default.json
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --plan-cache /tmp/pc2 > gpurun_out/bench_cachewrite.json 2>&1; echo "cache rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_launches_bench_n1024.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --plan-cache /tmp/pc2 > gpurun_out/ncu_bench.log 2>&1; echo "ncu rc=$?"
timeout 600 python scripts/stage_times.py --n 1024 > gpurun_out/r02_stage_times_n1024_chainkernel.jsonl 2>&1
BFSHT_CHAIN=0 timeout 600 python scripts/stage_times.py --n 1024 > gpurun_out/r02_stage_times_n1024_stagekernel.jsonl 2>&1
CACHE=/tmp/pc timeout 600 python scripts/chain_prof.py > gpurun_out/chain_plain.log 2>&1; tail -1 gpurun_out/chain_plain.log
CACHE=/tmp/pc timeout 900 ncu --set full --import-source on --clock-control none -k regex:alt_chain_kernel --launch-skip 6 --launch-count 5 -o gpurun_out/r02_chain_kernel -f python scripts/chain_prof.py > gpurun_out/ncu_chain.log 2>&1; tail -1 gpurun_out/ncu_chain.log
ncu -i gpurun_out/r02_chain_kernel.ncu-rep --page details --csv > gpurun_out/r02_ncu_chain_kernel_fwd_n1024_details.csv 2>/dev/null
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; tail -c 300 gpurun_out/bench_ref.json
