python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/traffic_plain.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --clock-control none -k regex:k_label -c 1 --csv --log-file gpurun_out/k_label_traffic_cfg5.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/traffic_ncu.log 2>&1
cat gpurun_out/k_label_traffic_cfg5.csv | tail -5
