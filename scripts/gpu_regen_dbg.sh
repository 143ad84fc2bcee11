python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1
for mode in full partial; do BFSHT_REGEN_COLS=$mode timeout 300 python scripts/regen_debug.py 128; done
bash scripts/gpu_regen2.sh 2>&1 | grep -v "^\.\|passed"
tail -2 gpurun_out/pytest_gpu.log
