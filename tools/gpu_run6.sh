python tools/ncu_target.py > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_sort|k_base' -o gpurun_out/r02_prof python tools/ncu_target.py > gpurun_out/ncu_run.log 2>&1
tail -5 gpurun_out/ncu_run.log
