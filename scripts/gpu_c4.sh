mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_fields.py 2>&1 | tail -2
timeout 900 python bench.py --workload c4 --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_c4.json').read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step'],2), round(d['roofline']['achieved'],2), round(d['roofline']['frac'],3), d.get('check_rel_l2_vs_oracle'))"
