mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_golden.py tests/test_gpu_n4096.py tests/test_gpu_sharded.py -q -x > gpurun_out/pytest_new.log 2>&1; tail -3 gpurun_out/pytest_new.log
python scripts/profile_step.py > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sht_ -c 2 -o gpurun_out/prof_dft256 python scripts/profile_step.py > gpurun_out/ncu_dft.log 2>&1
echo rc=$?
