# session-4 evidence: chain tests incl. regenerated plans, C4 with 3 groups
# x 2 slots, regeneration benches with the chain kernel, N=8192 chunk 0
mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_chain.py tests/test_gpu_fields.py tests/test_gpu_regen.py 2>&1 | tail -2
timeout 900 python bench.py --workload c4 --steps 5 --warmup 3 > gpurun_out/r02_bench_c4_group3x2_n1024.json 2> gpurun_out/bench_c4.err
python -c "
import json; d=json.loads(open('gpurun_out/r02_bench_c4_group3x2_n1024.json').read().strip().splitlines()[-1]); print('c4', round(d['value'],1), round(d['ms_per_step'],2), round(d['roofline']['achieved'],2), round(d['roofline']['frac'],3), d.get('check_rel_l2_vs_oracle'))"
for f in 1 0.5; do
  timeout 600 python bench.py --steps 10 --warmup 3 --regen $f --no-cpu-baseline > gpurun_out/r02_bench_n1024_regen${f}_chain.json 2> gpurun_out/bench_regen_$f.err
  python -c "
import json; d=json.loads(open('gpurun_out/r02_bench_n1024_regen${f}_chain.json').read().strip().splitlines()[-1]); r=d['roofline']; print('regen $f', round(d['value'],1), round(d['ms_per_step'],3), round(r['alt_fwd_ms'],3), round(r['alt_inv_ms'],3), d['roundtrip_rel_l2'])"
done
timeout 3000 python scripts/ooc_run.py --n 8192 --tol 1e-10 --chunks 48 --only 0 --decay 2 --real-grid --samples "" --rows 0,5000,8191 2> gpurun_out/ooc8192.err > gpurun_out/r02_ooc_n8192_chunk0_chain.json; tail -c 1200 gpurun_out/r02_ooc_n8192_chunk0_chain.json; tail -3 gpurun_out/ooc8192.err
