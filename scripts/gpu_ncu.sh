python scripts/ncu_label.py 5 300000 > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_label -s 1 -c 1 -o gpurun_out/prof_k_label python scripts/ncu_label.py 5 300000 > gpurun_out/ncu_full.log 2>&1
python scripts/ncu_label.py 5 300000 > gpurun_out/ncu_plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/ncu_label.py 5 300000 > gpurun_out/ncu_launch.log 2>&1
cat gpurun_out/ncu_plain.log; tail -5 gpurun_out/ncu_full.log
