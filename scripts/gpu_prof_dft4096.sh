mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:sht_synth_row --launch-skip 1 --launch-count 1 -o gpurun_out/synth4096_src -f python scripts/dft_stage_times.py --n 4096 > gpurun_out/ncu_s4096.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_s4096.log
