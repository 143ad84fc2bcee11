mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_graph.py tests/test_gpu_sht.py tests/test_gpu_fields.py tests/test_gpu_sharded.py tests/test_gpu_pipeline.py 2>&1 | tail -2
for v in graph nograph; do
  extra=""; [ $v = nograph ] && extra="--no-graph"
  timeout 600 python bench.py --warmup 3 --no-cpu-baseline $extra > gpurun_out/b_$v.json 2>gpurun_out/b_$v.err; python -c "
import json; d=json.loads(open('gpurun_out/b_$v.json').read().strip().splitlines()[-1]); print('$v', d['value'], d['ms_per_step'], d['e2e']['value'], d['gpu_launches'], d['roofline']['alt_fwd_ms'], d['roofline']['alt_inv_ms'])"
done
