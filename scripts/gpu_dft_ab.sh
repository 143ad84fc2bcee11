# DFT stage A/B: cluster row-pair kernels vs the one-CTA row-pair kernels
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
[ -n "$DFT_TESTS" ] && timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_sht.py tests/test_gpu_c2_parity.py tests/test_gpu_dft_big.py tests/test_gpu_pipeline.py tests/test_gpu_sharded.py tests/test_gpu_ooc.py 2>&1 | tail -3
for v in new legacy; do
  if [ $v = legacy ]; then export BFSHT_DFT_LEGACY=1; else unset BFSHT_DFT_LEGACY; fi
  echo "== $v"; timeout 600 python scripts/dft_stage_times.py --n ${DFT_NS:-1024,2048,4096} 2>&1 | tail -8
done
unset BFSHT_DFT_LEGACY
[ -n "$DFT_BENCH" ] && timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_dft.json 2> gpurun_out/bench_dft.err; tail -c 600 gpurun_out/bench_dft.json
