python tools/ncu_target.py normal > gpurun_out/ncu_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_base_big -c 1 -o gpurun_out/r02b_big python tools/ncu_target.py normal > gpurun_out/ncu_big.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sort -c 1 -o gpurun_out/r02b_sort python tools/ncu_target.py normal > gpurun_out/ncu_sort.log 2>&1
for r in big sort; do
  ncu -i gpurun_out/r02b_$r.ncu-rep --page raw --csv > gpurun_out/r02b_${r}_raw.csv 2>/dev/null
  ncu -i gpurun_out/r02b_$r.ncu-rep --page details > gpurun_out/r02b_${r}_details.txt 2>/dev/null
  ncu -i gpurun_out/r02b_$r.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r02b_${r}_source.csv 2>/dev/null
  gzip -9 gpurun_out/r02b_${r}_source.csv
done
for f in gpurun_out/r02b_*.ncu-rep; do gzip -9 $f; done
du -sh gpurun_out
