mkdir -p gpurun_out
ncu --version 2>&1 | tail -2
timeout 120 ncu --metrics gpu__time_duration.sum python -c "import torch; x=torch.zeros(4).cuda(); print(x.sum().item())" > gpurun_out/ncu_diag1.log 2>&1; echo "diag1 rc=$?"; tail -3 gpurun_out/ncu_diag1.log
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum -k regex:alt_stage -c 3 python scripts/profile_step.py --n 64 > gpurun_out/ncu_diag2.log 2>&1; echo "diag2 rc=$?"; tail -5 gpurun_out/ncu_diag2.log
