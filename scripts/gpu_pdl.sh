# programmatic dependent launch between the ALT stages: tests, then bench and
# per-direction ALT times with BFSHT_PDL=0 / 1
mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout 1200 python -m pytest -x -q -m gpu tests/test_gpu_chain.py tests/test_gpu_alt.py tests/test_gpu_golden.py tests/test_gpu_graph.py tests/test_gpu_sht.py tests/test_gpu_c2_parity.py tests/test_gpu_pipeline.py tests/test_gpu_sharded.py tests/test_gpu_regen.py 2>&1 | tail -2
for p in 1 0 1 0; do
  BFSHT_PDL=$p timeout 900 python bench.py --no-cpu-baseline --plan-cache /tmp/pc3 > gpurun_out/bench_pdl$p.json 2> gpurun_out/bench_pdl$p.err; echo "bench pdl=$p rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/bench_pdl$p.json').read().strip().splitlines()[-1]); print('pdl=$p', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['alt_fwd_ms'], d['roofline']['alt_inv_ms'], d['e2e']['value'], d.get('roundtrip_rel_l2'))"
done
