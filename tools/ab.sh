# A/B the default library against variants in build/var (bench K2 time + step)
mkdir -p gpurun_out
for lib in paper_1805_11775_b200/libhos_b200.so build/var/*.so; do
  [ -f "$lib" ] || continue
  HOS_LIB=$PWD/$lib python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/ab.log 2>&1
  tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$lib', 'step_ms %.4f'%d['ms_per_step'], 'k2_ms %.4f'%r['kernel_ms'], 'frac %.3f'%r['frac'], 'e2e_ms %.4f'%d['e2e']['ms_per_step'])" || tail -3 gpurun_out/ab.log
done
