# source-level ncu captures of the butterfly chain stages (N=1024 forward):
# stage 0 (gather tasks) and stage 3 (scatter tasks through lane maps)
mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
CACHE=/tmp/pc timeout 600 python scripts/chain_prof.py > gpurun_out/chain_plain.log 2>&1; tail -1 gpurun_out/chain_plain.log
CACHE=/tmp/pc timeout 900 ncu --set full --import-source on --clock-control none -k regex:alt_stage_kernel --launch-skip 7 --launch-count 4 -o gpurun_out/chain_src -f python scripts/chain_prof.py > gpurun_out/ncu_chain.log 2>&1; tail -2 gpurun_out/ncu_chain.log
ls -la gpurun_out
