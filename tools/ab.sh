# A/B: default library vs variant builds in build/var (tools/build_var.sh)
mkdir -p gpurun_out
run() {
  tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1', 'step_ms %.4f'%d['ms_per_step'], 'k2_ms %.4f'%r['kernel_ms'], 'frac %.3f'%r['frac'], 'e2e_ms %.4f'%d['e2e']['ms_per_step'], r.get('stage_us'))" || tail -3 gpurun_out/ab.log
}
python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-secondary > gpurun_out/ab.log 2>&1; run default
for lib in build/var/*.so; do
  [ -f "$lib" ] || continue
  HOS_LIB=$PWD/$lib python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-secondary > gpurun_out/ab.log 2>&1; run $lib
done
