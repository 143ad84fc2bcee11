mkdir -p gpurun_out
python -m paper_2004_11346_b200.build > gpurun_out/build.log 2>&1
timeout 600 python scripts/fields_step.py
timeout 900 ncu --target-processes application-only --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_fields.csv python scripts/fields_step.py > gpurun_out/ncu_fields.log 2>&1; echo "rc=$?"
