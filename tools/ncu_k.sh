# full ncu capture of one launch of kernel regex $2 on config $1
C=${1:-cfg2}; K=${2:-k_triple}
python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/prof_${K}_$C \
    python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ncu_k.log 2>&1
echo rc=$?
