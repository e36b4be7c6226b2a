python tools/ncu_target.py > gpurun_out/ncu_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_base_big -c 1 -o gpurun_out/r02_big python tools/ncu_target.py normal > gpurun_out/ncu_big.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sort -c 1 -o gpurun_out/r02_fb python tools/ncu_target.py fallback > gpurun_out/ncu_fb.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_base_wide -c 1 -o gpurun_out/r02_wide python tools/ncu_target.py c5 > gpurun_out/ncu_wide.log 2>&1
for r in big fb wide; do
  ncu -i gpurun_out/r02_$r.ncu-rep --page raw --csv > gpurun_out/r02_${r}_raw.csv 2>/dev/null
  ncu -i gpurun_out/r02_$r.ncu-rep --page details > gpurun_out/r02_${r}_details.txt 2>/dev/null
  ncu -i gpurun_out/r02_$r.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r02_${r}_source.csv 2>/dev/null
done
ls -la gpurun_out
du -sh gpurun_out
# keep the transfer under 64 MiB: drop the biggest artefacts first
for f in gpurun_out/r02_*_source.csv gpurun_out/r02_*.ncu-rep; do
  if [ $(du -sm gpurun_out | cut -f1) -gt 60 ]; then gzip -9 "$f"; fi
done
for f in gpurun_out/*.gz; do
  if [ $(du -sm gpurun_out | cut -f1) -gt 60 ]; then rm -f "$f"; fi
done
du -sh gpurun_out
