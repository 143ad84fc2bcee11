mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
export F=64 CACHE=/tmp/fc
timeout 600 python scripts/fields_step.py 2>&1 | tail -1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:alt_group_kernel --launch-skip 6 --launch-count 1 -o gpurun_out/group_src -f python scripts/fields_step.py > gpurun_out/ncu_group.log 2>&1; echo ncu rc=$?; tail -2 gpurun_out/ncu_group.log
