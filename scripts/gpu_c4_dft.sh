# group engine (C4) + row/scratch DFT kernels: tests, A/B timings, C4 bench
mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_fields.py tests/test_gpu_sht.py tests/test_gpu_c2_parity.py tests/test_gpu_dft_big.py tests/test_gpu_pipeline.py tests/test_gpu_sharded.py tests/test_gpu_ooc.py 2>&1 | tail -3
for v in current; do
  echo "== $v"; timeout 600 python scripts/dft_stage_times.py --n ${DFT_NS:-1024,2048,4096} 2>&1 | grep '"kernel"' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['n'], d['kernel'], round(d['ms'],4), round(d['frac_of_peak'],3))"
done
for v in group wide16; do
  unset BFSHT_FIELDS_WIDE16; [ $v = wide16 ] && export BFSHT_FIELDS_WIDE16=1
  timeout 900 python bench.py --workload c4 --steps 5 --warmup 3 > gpurun_out/bench_c4_$v.json 2> gpurun_out/bench_c4_$v.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_c4_$v.json').read().strip().splitlines()[-1]); print('$v', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'], d.get('check_vs_oracle', d.get('parity')))"
done
timeout 900 python scripts/plan_times.py --n 4096 --orders 64 > gpurun_out/plan_times_n4096.json 2> gpurun_out/plan_times.err; echo plan rc=$?; cat gpurun_out/plan_times_n4096.json
