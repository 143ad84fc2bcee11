mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x -k "batch or io or cache or sht" > gpurun_out/pytest_batch.log 2>&1; tail -2 gpurun_out/pytest_batch.log
for b in 2 4; do
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --batch $b > gpurun_out/bench_batch$b.json 2> gpurun_out/bench_batch$b.err; echo "batch $b rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_batch$b.json').read().strip().splitlines()[-1]); r=d['roofline']; print($b, round(d['value'],1), round(d['ms_per_step'],3), round(r['alt_fwd_ms'],3), round(r['alt_inv_ms'],3), round(r['frac'],3), round(d['e2e']['value'],1), d['roundtrip_rel_l2'])"
done
