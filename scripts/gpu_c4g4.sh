# group engine G=4 (64 fields per pass) vs G=2 (32) vs 16-wide (8); e2e vs steps
mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_fields.py 2>&1 | tail -2
for v in g4 g2; do
  unset BFSHT_FIELDS_GROUP64; [ $v = g2 ] && export BFSHT_FIELDS_GROUP64=1
  timeout 900 python bench.py --workload c4 --steps 5 --warmup 3 > gpurun_out/bench_c4_$v.json 2> gpurun_out/bench_c4_$v.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_c4_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['value'],1), round(d['ms_per_step'],2), round(d['roofline']['achieved'],2), round(d['roofline']['frac'],3), d.get('parity'))"
done
unset BFSHT_FIELDS_GROUP64
timeout 600 python bench.py --steps 50 --warmup 3 --no-cpu-baseline > gpurun_out/bench_s50.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/bench_s50.json').read().strip().splitlines()[-1]); print('steps50', d['value'], d['e2e']['value'])"
