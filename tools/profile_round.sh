# Round profile capture (1 GPU): plain bench, launch list, full ncu of the
# triple-product kernel.  Outputs in gpurun_out/; summaries go to profiles/.
set -e
mkdir -p gpurun_out
python bench.py --steps 200 --warmup 10 > gpurun_out/bench_full.log 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_triple -s 2 -c 1 -o gpurun_out/prof_triple \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_line_scan -s 2 -c 1 -o gpurun_out/prof_scan \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu3.log 2>&1
echo profile-done
