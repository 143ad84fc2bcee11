# chain kernel: bundle / cost-model sweep (per-stage times), then a
# source-level ncu capture of the forward chain stages at N=1024
mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
summ() {
python - "$1" <<'PY'
import json, sys
rows=[json.loads(l) for l in open(sys.argv[1]) if l.startswith('{')]
ch=[r for r in rows if r['tile_MB']<5000]
print(sys.argv[1].split('/')[-1], 'chain ms', round(sum(r['ms'] for r in ch),4), [round(r['ms'],3) for r in ch])
PY
}
for cfg in ${SWEEP:-"6 3072" "1 3072" "3 3072" "12 3072" "6 1024" "6 8192"}; do
  set -- $cfg
  BFSHT_CHAIN_BUNDLES=$1 BFSHT_CHAIN_CFIX=$2 timeout 600 python scripts/stage_times.py --n 1024 > gpurun_out/st_b$1_c$2.jsonl 2>&1
  summ gpurun_out/st_b$1_c$2.jsonl
done
CACHE=/tmp/pc timeout 600 python scripts/chain_prof.py > gpurun_out/chain_plain.log 2>&1; tail -1 gpurun_out/chain_plain.log
CACHE=/tmp/pc timeout 900 ncu --set full --import-source on --clock-control none -k regex:alt_chain_kernel --launch-skip 6 --launch-count 5 -o gpurun_out/chain_src2 -f python scripts/chain_prof.py > gpurun_out/ncu_chain.log 2>&1; tail -2 gpurun_out/ncu_chain.log
