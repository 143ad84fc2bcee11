# regen v6 (straight-line full tiles): bitwise tests, then the N=1024 bench at several fractions
mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_regen.py 2>&1 | tail -2
for f in 1 0.5 0.3 0; do
  timeout 600 python bench.py --steps 10 --warmup 3 --regen $f --no-cpu-baseline > gpurun_out/bench_regen_$f.json 2> gpurun_out/bench_regen_$f.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_regen_$f.json').read().strip().splitlines()[-1]); r=d['roofline']; print('regen $f', round(d['value'],1), round(d['ms_per_step'],3), round(r['alt_fwd_ms'],3), round(r['alt_inv_ms'],3), d['roundtrip_rel_l2'])"
done
