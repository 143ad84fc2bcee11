mkdir -p gpurun_out
for cfg in "12 2" "8 3" "6 4"; do
  set -- $cfg
  BFSHT_NVCC_FLAGS="-DBF_WARPS=$1 -DBF_STAGES=$2" python -m paper_2004_11346_b200.build --force > gpurun_out/build_$1_$2.log 2>&1 || { echo "build $1x$2 failed"; continue; }
  timeout 600 python scripts/stage_times.py --reps 5 > gpurun_out/st_$1_$2.jsonl 2>/dev/null
  python -c "
import json
r=[json.loads(l) for l in open('gpurun_out/st_$1_$2.jsonl')]
ch=sum(d['ms'] for d in r if d['tile_MB']<3000); fin=sum(d['ms'] for d in r if d['tile_MB']>=3000)
print('$1 warps x $2 slots: chain %.3f ms, final %.3f ms (fwd+inv)'%(ch,fin))"
done
python -m paper_2004_11346_b200.build --force > gpurun_out/build.log 2>&1
