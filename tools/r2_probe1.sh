set -x
nproc; free -g; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
python -c "import paper_1305_3122_b200.build as b; b.build()"
timeout 300 python tools/quick_time.py C1 C2 C3 C4 > gpurun_out/p1_quick.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p1_launch_C5.csv python tools/profile_once.py C5 2 > gpurun_out/p1_ncu_C5.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_rows -c 1 -o gpurun_out/p1_rows_C3 python tools/profile_once.py C3 1 > gpurun_out/p1_ncu_C3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_rows -c 1 -o gpurun_out/p1_rows_C5 python tools/profile_once.py C5 1 > gpurun_out/p1_ncu_C5full.log 2>&1
ls -la gpurun_out
