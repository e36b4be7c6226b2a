#!/bin/bash
# Round measurement on the GPU box: bench line (ours + reference arm), launch list of the same bench
# command, one ncu --set full capture of k_sort and k_base_big, summaries -> gpurun_out/.
#   gpurun --timeout 1500 -- 'bash tools/measure.sh'
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out
mkdir -p $O
timeout 400 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 300 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "bench ref rc=$?"
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $O/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_sort|k_base_big" -c 2 -f -o $O/full \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py $O/ncu_kernels.json $O/full.ncu-rep > /dev/null; echo "summary rc=$?"
tail -c 600 $O/bench.json
