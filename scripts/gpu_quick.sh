python scripts/ncu_aux.py 3 > gpurun_out/aux_plain.log 2>&1 && \
ncu --set full --clock-control none -k regex:"k_fixup|k_label_tets" -c 2 -o gpurun_out/prof_aux python scripts/ncu_aux.py 3 > gpurun_out/aux_ncu.log 2>&1
cat gpurun_out/aux_plain.log; tail -2 gpurun_out/aux_ncu.log
