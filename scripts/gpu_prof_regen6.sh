mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
ls -la /tmp | grep -i nsight; ncu --version | tail -1
rm -rf /tmp/nsight-compute-lock /tmp/nsight* 2>/dev/null
mkdir -p /tmp/ncu_tmp; export TMPDIR=/tmp/ncu_tmp
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:alt_stage_kernel --launch-skip 6 --launch-count 1 -o gpurun_out/regen6_src -f python scripts/profile_step.py --regen 1 > gpurun_out/ncu_regen6.log 2>&1; echo ncu rc=$?; tail -2 gpurun_out/ncu_regen6.log
