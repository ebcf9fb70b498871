# K2 kernel choice A/B on one config: k_triple_cta (default) vs HOS_K2=warp
#   tools/k2_ab.sh cfg3 [steps]
c=${1:-cfg3}; n=${2:-20}
mkdir -p gpurun_out
run() {
  tail -1 gpurun_out/k2ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline'] or {}; print('$c $1', 'step_ms %.4f'%d['ms_per_step'], 'frac', r.get('frac'), r.get('kernel'), r.get('stage_us'))" || tail -3 gpurun_out/k2ab.log
}
for rep in 1 2; do
  timeout 200 python bench.py --config $c --steps $n --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/k2ab.log 2>&1; run cta
  HOS_K2=warp timeout 200 python bench.py --config $c --steps $n --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/k2ab.log 2>&1; run warp
done
