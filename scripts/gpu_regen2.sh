mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x  > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for f in 0 0.25 0.5 1.0; do
  timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --regen $f > gpurun_out/bench_regen_$f.json 2> gpurun_out/bench_regen_$f.err; echo "regen $f rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/bench_regen_$f.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$f', round(d['value'],1), round(d['ms_per_step'],3), round(r['alt_fwd_ms'],3), round(r['alt_inv_ms'],3), round(r['frac'],3), round(d['e2e']['value'],1), d['roundtrip_rel_l2'], r.get('regen',{}).get('hbm_GBps_rank0'))"
done
