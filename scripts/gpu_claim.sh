mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
for k in 1 2 4 8; do
  BFSHT_CLAIM=$k timeout 600 python scripts/stage_times.py --reps 5 > gpurun_out/st_claim$k.jsonl 2>/dev/null
  python -c "
import json
r=[json.loads(l) for l in open('gpurun_out/st_claim$k.jsonl')]
ch=sum(d['ms'] for d in r if d['tile_MB']<3000); fin=sum(d['ms'] for d in r if d['tile_MB']>=3000)
print('claim $k: chain %.3f ms, final %.3f ms (fwd+inv)'%(ch,fin))"
done
