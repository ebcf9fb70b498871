# Round-2 profile capture (1 GPU): launch list of the cfg2 bench and full ncu
# captures of the top kernels per config.  Outputs gpurun_out/r02_*.
set -x
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-secondary"
$B > gpurun_out/r02_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv $B > gpurun_out/r02_ncu_l.log 2>&1
for spec in "cfg2:k_triple" "cfg2:k_front" "cfg2:k_line_scan" "cfg2:k_box3" "cfg3:k_triple" "cfg4:k_triple" "cfg5:k_triple" "cfg5:k_smooth_series_sep" "cfg5:k_front"; do
  c=${spec%%:*}; k=${spec##*:}
  python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/r02_plain_$c.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/r02_prof_${k}_$c \
      python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/r02_ncu_${k}_$c.log 2>&1
done
echo profile-done
# summarise on the box (the reports are too large to bring back together)
for f in gpurun_out/r02_prof_*.ncu-rep; do
  b=$(basename $f .ncu-rep)
  python tools/ncu_summary.py $f > gpurun_out/${b}.txt 2>&1
  ncu -i $f --page raw --csv > gpurun_out/${b}_raw.csv 2>/dev/null
  gzip -f gpurun_out/${b}_raw.csv
done
mkdir -p gpurun_out/keep && mv gpurun_out/r02_prof_k_triple_cfg2.ncu-rep gpurun_out/r02_prof_k_smooth_series_sep_cfg5.ncu-rep gpurun_out/keep/ 2>/dev/null
rm -f gpurun_out/r02_prof_*.ncu-rep
mv gpurun_out/keep/* gpurun_out/ && rmdir gpurun_out/keep
ls -la gpurun_out | tail -40
