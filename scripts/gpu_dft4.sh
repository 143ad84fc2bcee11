mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python scripts/dft_times.py 2>&1 | tail -1
timeout 600 python scripts/dft_big_times.py 2>&1 | tail -2
