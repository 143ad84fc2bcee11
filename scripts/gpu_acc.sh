mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout 600 python scripts/stage_times.py --reps 5 > gpurun_out/st_acc.jsonl 2>/dev/null
python -c "
import json
r=[json.loads(l) for l in open('gpurun_out/st_acc.jsonl')]
ch=sum(d['ms'] for d in r if d['tile_MB']<3000); fin=sum(d['ms'] for d in r if d['tile_MB']>=3000)
print('split acc: chain %.3f ms, final %.3f ms (fwd+inv)'%(ch,fin))"
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_acc.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/bench_acc.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['roundtrip_rel_l2'])"
