# source-level ncu captures: butterfly chain stages 0-1 (N=1024 forward) and
# the cluster row-pair DFT synthesis kernel (N=1024)
mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout 600 python scripts/stage_times.py --n 1024 > gpurun_out/stage_times_n1024.jsonl 2>&1; tail -3 gpurun_out/stage_times_n1024.jsonl
timeout 900 ncu --set full --import-source on --clock-control none -k regex:alt_stage_kernel --launch-skip 7 --launch-count 4 -o gpurun_out/chain_src -f python scripts/chain_prof.py > gpurun_out/ncu_chain.log 2>&1; tail -2 gpurun_out/ncu_chain.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:sht_synth_pair --launch-skip 2 --launch-count 1 -o gpurun_out/synth_src -f python scripts/dft_stage_times.py --n 1024 > gpurun_out/ncu_synth.log 2>&1; tail -2 gpurun_out/ncu_synth.log
ls -la gpurun_out
