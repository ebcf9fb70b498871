# Round profile capture (1 GPU): plain bench, launch list, full ncu of each
# pipeline kernel.  Outputs in gpurun_out/; tools/make_profiles.py writes the
# summaries under profiles/.
set -e
mkdir -p gpurun_out
python bench.py --steps 200 --warmup 10 > gpurun_out/bench_full.log 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ncu1.log 2>&1
for k in k_triple k_front k_line_scan k_box3; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_$k \
      python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ncu_$k.log 2>&1
done
echo profile-done
