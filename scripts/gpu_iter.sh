mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python scripts/stage_times.py > gpurun_out/stages.jsonl 2> gpurun_out/stages.err; echo rc=$?
python - <<'PY'
import json
for l in open("gpurun_out/stages.jsonl"):
    r = json.loads(l); print(r["dir"], r["stage"], r["tasks"], r["ops"], round(r["avg_tile_KB"],2), round(r["ms"],4), round(r["tile_GBps"]))
PY
tail -3 gpurun_out/stages.err
