# Timing-only experiment (round 1): BFSHT_DEBUG_DROP_ADDS was a temporary packer patch
# (drop every index-add op; wrong results) that is not in the tree any more.
mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1
timeout 600 python scripts/stage_times.py --reps 5 > gpurun_out/st_base.jsonl 2>/dev/null
BFSHT_DEBUG_DROP_ADDS=1 timeout 600 python scripts/stage_times.py --reps 5 > gpurun_out/st_noadd.jsonl 2>/dev/null
for f in base noadd; do python -c "
import json
r=[json.loads(l) for l in open('gpurun_out/st_$f.jsonl')]
ch=sum(d['ms'] for d in r if d['tile_MB']<3000); fin=sum(d['ms'] for d in r if d['tile_MB']>=3000)
print('$f: chain %.3f ms, final %.3f ms, ops %d'%(ch,fin,sum(d['ops'] for d in r)))"; done
