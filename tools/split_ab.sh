for sp in 1:1 21:19 22:18 23:17 24:16 25:15; do
  HOS_K2_SPLIT=$sp python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-secondary > gpurun_out/ab.log 2>&1
  tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$sp', 'step %.4f'%d['ms_per_step'], 'k2 %.4f'%r['kernel_ms'], r['stage_us'])"
done
