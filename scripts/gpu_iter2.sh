mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python scripts/stage_times.py > gpurun_out/stages.jsonl 2> gpurun_out/stages.err; echo rc=$?
python - <<'PY'
import json
for l in open("gpurun_out/stages.jsonl"):
    r = json.loads(l); print(r["dir"], r["stage"], r["tasks"], r["ops"], round(r["avg_tile_KB"],2), round(r["ms"],4), round(r["tile_GBps"]))
PY
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['alt_fwd_ms'], d['roofline']['alt_inv_ms'], d['roofline']['frac'], d['e2e']['value'], d['roundtrip_rel_l2'])"
