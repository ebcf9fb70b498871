# Final round-2 profile capture (1 GPU): launch list of the default bench and
# full ncu captures of the top kernels per config, summarised on the box.
# Outputs gpurun_out/fin_*.
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-secondary"
$B > gpurun_out/fin_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fin_launches.csv $B > gpurun_out/fin_ncu_l.log 2>&1
for spec in "cfg2:k_triple" "cfg2:k_front" "cfg2:k_raw_cells" "cfg2:k_box_tiles" "cfg3:k_triple" "cfg4:k_triple" "cfg5:k_triple" "cfg5:k_smooth_series_pipe" "cfg5:k_front_r16"; do
  c=${spec%%:*}; k=${spec##*:}
  python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/fin_plain_$c.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/fin_prof_${k}_$c \
      python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/fin_ncu_${k}_$c.log 2>&1
  f=gpurun_out/fin_prof_${k}_$c.ncu-rep
  if [ -f $f ]; then
    python tools/ncu_summary.py $f > gpurun_out/fin_${k}_$c.txt 2>&1
    rm -f $f
  fi
done
ls -la gpurun_out | tail -30
