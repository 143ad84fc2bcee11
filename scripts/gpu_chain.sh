# chain kernel: bitwise tests, then per-stage times and the bench with the
# chain kernel off (BFSHT_CHAIN=0) and on (default)
mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout 900 python -m pytest tests/test_gpu_chain.py tests/test_gpu_alt.py tests/test_gpu_sht.py tests/test_gpu_golden.py -x -q > gpurun_out/pytest_chain.log 2>&1; tail -15 gpurun_out/pytest_chain.log
for c in ${CHAIN_MODES:-0 1}; do
  BFSHT_CHAIN=$c timeout 600 python scripts/stage_times.py --n 1024 > gpurun_out/stage_times_n1024_chain$c.jsonl 2>&1
  python - <<PY
import json
rows=[json.loads(l) for l in open('gpurun_out/stage_times_n1024_chain$c.jsonl') if l.startswith('{')]
ch=[r for r in rows if r['tile_MB']<5000]
print('chain=$c chain-stage ms', round(sum(r['ms'] for r in ch),4), 'final ms', round(sum(r['ms'] for r in rows if r['tile_MB']>=5000),4), [round(r['ms'],3) for r in rows])
PY
done
for c in ${CHAIN_MODES:-0 1}; do
  BFSHT_CHAIN=$c timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_chain$c.json 2> gpurun_out/bench_chain$c.err; echo "bench chain=$c rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/bench_chain$c.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['alt_fwd_ms'], d['roofline']['alt_inv_ms'], d['e2e']['value'], d.get('roundtrip_rel_l2'))"
done
