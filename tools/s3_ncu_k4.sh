B="python bench.py --config cfg2 --steps 3 --warmup 3 --no-cpu-baseline --no-secondary"
$B > gpurun_out/k4n_plain.log 2>&1 || exit 1
for k in k_raw_cells k_box_tiles; do
ncu --set full --clock-control none --cache-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/k4n_$k $B > gpurun_out/k4n_ncu_$k.log 2>&1
python tools/ncu_summary.py gpurun_out/k4n_$k.ncu-rep > gpurun_out/k4n_$k.txt 2>&1
ncu -i gpurun_out/k4n_$k.ncu-rep --page details > gpurun_out/k4n_${k}_details.txt 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 60 --csv --log-file gpurun_out/k4n_launches.csv $B > gpurun_out/k4n_l.log 2>&1
echo done
