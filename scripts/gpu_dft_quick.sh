mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_dft_big.py tests/test_gpu_sht.py tests/test_gpu_c2_parity.py tests/test_gpu_golden.py tests/test_gpu_sharded.py tests/test_gpu_ooc.py 2>&1 | tail -1
timeout 600 python scripts/dft_stage_times.py --n ${DFT_NS:-1024,4096} 2>&1 | grep '"kernel"' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['n'], d['kernel'], round(d['ms'],4), round(d['frac_of_peak'],3))"
timeout 600 python bench.py --warmup 3 --no-cpu-baseline --plan-cache /tmp/pc > gpurun_out/b_q.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/b_q.json').read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step'],4), round(d['e2e']['value'],1), d['roundtrip_rel_l2'])"
