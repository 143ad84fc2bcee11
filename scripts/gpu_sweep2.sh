# bundle-count sweep for the chain kernel (N=1024 per-stage times) and the
# DFT stage alone at N = 1024 / 4096
mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
for b in 8 16 32 1000; do
  BFSHT_CHAIN_BUNDLES=$b timeout 600 python scripts/stage_times.py --n 1024 > gpurun_out/st_b$b.jsonl 2>&1
  python - $b <<'PY'
import json, sys
rows=[json.loads(l) for l in open(f'gpurun_out/st_b{sys.argv[1]}.jsonl') if l.startswith('{')]
ch=[r for r in rows if r['tile_MB']<5000]
print('bundles/warp', sys.argv[1], 'chain ms', round(sum(r['ms'] for r in ch),4), [round(r['ms'],3) for r in ch])
PY
done
timeout 600 python scripts/dft_stage_times.py --n 1024,4096 2>&1 | grep '"kernel"' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['n'], d['kernel'], round(d['ms'],4), round(d['frac_of_peak'],3))"
