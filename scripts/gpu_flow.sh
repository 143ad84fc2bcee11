mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -q -m gpu -x -k "flow" > gpurun_out/pytest_flow.log 2>&1; tail -3 gpurun_out/pytest_flow.log
GAPS=1776,3552,8000 timeout 900 python scripts/flow_times.py 2> gpurun_out/flow.err | tee gpurun_out/flow_times.jsonl
tail -3 gpurun_out/flow.err
