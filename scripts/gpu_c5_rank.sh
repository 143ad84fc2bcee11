# C5 at the rank level: one eighth of the N=8192 orders (6 of 48 LPT chunks,
# the share of one rank at P=8) planned with every full-height turning tile
# regenerated (f1), kept resident on one B200 between the forward and the
# inverse; config-5 inputs ((1+k)^-2 coefficients, real U(-1,1) grid)
mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; exit 1; }
rm -f /dev/shm/bfsht_plan_*
# small first: the same path at N=64 with regeneration (must pass its checks)
timeout 600 python scripts/ooc_run.py --n 64 --tol 1e-12 --chunks 4 --only 0,2 --regen 1 --decay 2 --real-grid --samples "" --rows 0,10,63 --out gpurun_out/ooc_small_regen.json 2> gpurun_out/ooc_small_regen.err | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('small', d['checks'], d['resident_chunks_after_forward'])" || { tail -20 gpurun_out/ooc_small_regen.err; exit 1; }
( while true; do free -g | sed -n 2p; nvidia-smi --query-gpu=memory.used --format=csv,noheader; sleep 60; done ) > gpurun_out/c5_mem.log 2>&1 &
timeout 3300 python scripts/ooc_run.py --n 8192 --tol 1e-10 --chunks 48 --only 0,8,16,24,32,40 --regen 1 --decay 2 --real-grid --reserve-gb 6 --rows 0,4000,8191 --out gpurun_out/c5_rank_regen.json 2> gpurun_out/c5_rank.err | tail -c 2500; echo rc=$?; tail -12 gpurun_out/c5_rank.err
