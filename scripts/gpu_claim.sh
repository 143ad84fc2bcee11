# task-claim shards A/B: BF_CLAIM_SHARDS=4 (default) vs 1 (one counter per stage)
mkdir -p gpurun_out
for k in 4 1 8; do
  touch paper_2004_11346_b200/csrc/*.cu
  BFSHT_NVCC_FLAGS="-DBF_CLAIM_SHARDS=$k" python -m paper_2004_11346_b200.build > gpurun_out/build_$k.log 2>&1 || { tail -5 gpurun_out/build_$k.log; exit 1; }
  [ $k = 4 ] && timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_sht.py tests/test_gpu_fields.py tests/test_gpu_golden.py tests/test_gpu_alt.py 2>&1 | tail -1
  timeout 600 python bench.py --warmup 3 --no-cpu-baseline --plan-cache /tmp/pc > gpurun_out/b_claim$k.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/b_claim$k.json').read().strip().splitlines()[-1]); print('shards $k', round(d['value'],1), round(d['ms_per_step'],4), round(d['roofline']['alt_fwd_ms'],4), round(d['roofline']['alt_inv_ms'],4), round(d['e2e']['value'],1))"
  timeout 600 python scripts/stage_times.py --n 1024 2>/dev/null | python -c "
import sys,json
tot={0:0,1:0}
for l in sys.stdin:
    try: d=json.loads(l)
    except: continue
    if d['tile_MB']<5000: tot[d['dir']]+=d['ms']
print('  chain ms fwd/inv', round(tot[0],4), round(tot[1],4))"
done
