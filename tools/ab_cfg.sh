# A/B on one config: default library vs variant builds in build/var
#   tools/ab_cfg.sh cfg5 [steps]
c=${1:-cfg5}; n=${2:-20}
mkdir -p gpurun_out
run() {
  tail -1 gpurun_out/abc.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline'] or {}; print('$c $1', 'step_ms %.4f'%d['ms_per_step'], 'frac', r.get('frac'), r.get('in_step_us'))" || tail -3 gpurun_out/abc.log
}
for rep in 1 2; do
timeout 150 python bench.py --config $c --steps $n --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/abc.log 2>&1; run default
for lib in build/var/*.so; do
  [ -f "$lib" ] || continue
  HOS_LIB=$PWD/$lib timeout 150 python bench.py --config $c --steps $n --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/abc.log 2>&1; run $lib
done
done
