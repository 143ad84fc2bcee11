mkdir -p gpurun_out
for t in 256 384 512; do
  BFSHT_NVCC_FLAGS="-DBF_DFT_THREADS=$t" python -m paper_2004_11346_b200.build --force > gpurun_out/build_$t.log 2>&1
  timeout 600 python scripts/dft_times.py >> gpurun_out/dft_times.jsonl 2> gpurun_out/dft_$t.err; echo "t=$t rc=$?"
done
cat gpurun_out/dft_times.jsonl
