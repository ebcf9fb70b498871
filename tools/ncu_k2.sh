# full ncu capture of one K2 launch (cfg given as $1, default cfg2)
C=${1:-cfg2}
python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_triple -s 4 -c 1 -o gpurun_out/prof_k2_$C \
    python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ncu_k2.log 2>&1
echo rc=$?
