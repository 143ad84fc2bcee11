# DMMA generic-radix butterflies: DFT tests + stage times
mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_dft_big.py tests/test_gpu_sht.py tests/test_gpu_c2_parity.py tests/test_gpu_ooc.py tests/test_gpu_n4096.py 2>&1 | tail -3
timeout 600 python scripts/dft_stage_times.py --n 1024,2048,4096,8192 2>&1 | grep '"kernel"' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['n'], d['kernel'], round(d['ms'],4), round(d['frac_of_peak'],3))"
