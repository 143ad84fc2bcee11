# whole SHT at N=2048 on one GPU through the chunked runner (the whole plan
# does not fit the host's RAM at once): L = 8191 is prime, so every phi row
# is a Bluestein row; oracle (numpy pocketfft) on every order
mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; exit 1; }
timeout 3000 python scripts/ooc_run.py --n 2048 --tol 1e-12 --chunks 8 --samples 0,1,1024,3000,4095 --oracle-all 2> gpurun_out/ooc2048.err > gpurun_out/r02_ooc_n2048.json; echo rc=$?
tail -c 1800 gpurun_out/r02_ooc_n2048.json; tail -4 gpurun_out/ooc2048.err
