# per-stage ALT times of one N=4096 chunk (1/24 of the orders, tol 1e-10)
# with the chain kernel off and on
mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
for c in 0 1; do
  BFSHT_CHAIN=$c timeout 1500 python scripts/stage_times.py --n 4096 --tol 1e-10 --chunk 24 > gpurun_out/stage_times_n4096_chunk_chain$c.jsonl 2>&1
  python - <<PY
import json
rows=[json.loads(l) for l in open('gpurun_out/stage_times_n4096_chunk_chain$c.jsonl') if l.startswith('{')]
for d in (0,1):
    rr=[r for r in rows if r['dir']==d]
    fin=max(rr,key=lambda r:r['tile_MB'])
    ch=[r for r in rr if r is not fin]
    tb=sum(r['tile_MB'] for r in ch); ms=sum(r['ms'] for r in ch)
    print('chain=$c dir',d,'chain ms',round(ms,3),'chain tile GB',round(tb/1e3,2),'TB/s',round(tb/ms/1e6,2),'final ms',round(fin['ms'],3),'final TB/s',round(fin['tile_GBps']/1e3,2),'all ms',round(ms+fin['ms'],3),'all tile TB/s', round((tb+fin['tile_MB'])/(ms+fin['ms'])/1e6,2))
PY
done
