# round-2 evidence snapshot: bench lines, reference arm, launch list, ncu of the leaf kernels
python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
python bench.py --impl reference > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_reference.err
python bench.py --config C5 --steps 5 --warmup 2 --no-cpu > gpurun_out/r02_bench_C5.json 2> gpurun_out/r02_bench_C5.err
python bench.py --no-e2e --no-cpu --steps 2 --warmup 1 > gpurun_out/r02_launch_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv python bench.py --no-e2e --no-cpu --steps 2 --warmup 1 > gpurun_out/r02_launch_ncu.log 2>&1
python tools/ncu_target.py c5 > gpurun_out/ncu_plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_base_wide -c 1 -o gpurun_out/r02c_wide python tools/ncu_target.py c5 > gpurun_out/ncu_wide.log 2>&1
ncu -i gpurun_out/r02c_wide.ncu-rep --page raw --csv > gpurun_out/r02c_wide_raw.csv 2>/dev/null
ncu -i gpurun_out/r02c_wide.ncu-rep --page details > gpurun_out/r02c_wide_details.txt 2>/dev/null
ncu -i gpurun_out/r02c_wide.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r02c_wide_source.csv 2>/dev/null
gzip -9 gpurun_out/r02c_wide_source.csv gpurun_out/r02c_wide.ncu-rep
du -sh gpurun_out
