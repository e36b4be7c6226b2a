# round-2 evidence snapshot (after the last kernel change): tests, smoke, bench lines (R, reference arm,
# C5, C1, the C2 patterns), config table, launch list, ncu --set full of the kernels
#   gpurun --timeout 3000 -- 'bash tools/gpu_snap.sh'
O=gpurun_out
mkdir -p $O
python -m pytest tests -m gpu -q > $O/r02_gpu_tests.log 2>&1; tail -2 $O/r02_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/r02_smoke.log 2>&1; tail -c 200 $O/r02_smoke.log
python bench.py > $O/r02_bench.json 2> $O/r02_bench.err; echo "bench rc=$?"
python bench.py --impl reference > $O/r02_bench_reference.json 2> $O/r02_bench_reference.err; echo "ref rc=$?"
python bench.py --config C5 --steps 5 --warmup 3 --no-cpu > $O/r02_bench_C5.json 2> $O/r02_bench_C5.err; echo "C5 rc=$?"
: > $O/r02_bench_configs.jsonl
for c in C1 C2.asc C2.desc C2.organ C2.asc_tail C2.asc_swaps; do
  python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e >> $O/r02_bench_configs.jsonl 2>> $O/r02_bench_configs.err
done
python tools/config_times.py > $O/r02_config_times.md 2>&1
python tools/runs_prof.py > $O/r02_runs_prof.log 2>&1
python tools/small_n.py 2>&1 | grep '"depth_limit": 0' > $O/r02_small_n.log
python bench.py --no-e2e --no-cpu --steps 2 --warmup 3 > $O/r02_launch_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r02_launches.csv python bench.py --no-e2e --no-cpu --steps 2 --warmup 3 > $O/r02_launch_ncu.log 2>&1
python tools/ncu_target.py normal > $O/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_sort|k_base_big' -c 2 -f -o $O/r02_full python tools/ncu_target.py normal > $O/ncu_full.log 2>&1
python tools/ncu_target.py c5 > $O/ncu_plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_base_wide -c 1 -f -o $O/r02_wide python tools/ncu_target.py c5 > $O/ncu_wide.log 2>&1
python tools/runs_prof.py 24 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_base_big|k_check' -c 4 -f -o $O/r02_runs python tools/ncu_target.py organ > $O/ncu_runs.log 2>&1
python tools/ncu_summary.py $O/r02_ncu_kernels.json $O/r02_full.ncu-rep $O/r02_wide.ncu-rep > /dev/null 2>&1
python tools/ncu_summary.py $O/r02_ncu_runs_kernels.json $O/r02_runs.ncu-rep > /dev/null 2>&1
for r in full wide runs; do
  ncu -i $O/r02_$r.ncu-rep --page details > $O/r02_ncu_${r}_details.txt 2>/dev/null
  ncu -i $O/r02_$r.ncu-rep --page source --csv --print-source cuda,sass > $O/r02_${r}_source.csv 2>/dev/null
  gzip -9f $O/r02_${r}_source.csv
done
rm -f $O/r02_*.ncu-rep
du -sh $O
