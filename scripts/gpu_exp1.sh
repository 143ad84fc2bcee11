# experiments: Bluestein vs direct mixed radix for long rows; group-engine ncu
mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
for v in direct blue; do
  unset BFSHT_BLUESTEIN_ABOVE; [ $v = blue ] && export BFSHT_BLUESTEIN_ABOVE=13
  echo "== $v"; timeout 600 python scripts/dft_stage_times.py --n 4096,8192 2>&1 | grep '"kernel"' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['n'], d['kernel'], round(d['ms'],4), round(d['frac_of_peak'],3))"
done
unset BFSHT_BLUESTEIN_ABOVE
timeout 900 ncu --set full --import-source on --clock-control none -k regex:alt_group_kernel --launch-skip 6 --launch-count 1 -o gpurun_out/group_src -f env F=64 python scripts/fields_step.py > gpurun_out/ncu_group.log 2>&1; tail -2 gpurun_out/ncu_group.log
