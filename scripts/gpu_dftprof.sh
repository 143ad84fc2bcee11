mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1
timeout 600 ncu --target-processes application-only --set full --clock-control none --import-source on -k regex:dft_rows -c 1 -o gpurun_out/prof_dft16383 python scripts/dft_prof.py 16383 2368 > gpurun_out/ncu_dft.log 2>&1; echo rc=$?; tail -2 gpurun_out/ncu_dft.log
