# K2 tile step A/B: parity under each forced step, then the configs bench per step
set -x
mkdir -p gpurun_out
for t in 2 4; do
  HOS_K2_TILE=$t timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
done
for t in 4 2; do
  echo "== HOS_K2_TILE=$t"
  HOS_K2_TILE=$t bash tools/configs_bench.sh ${@:-cfg2 cfg4 cfg5 cfg3}
done
echo "== auto"
bash tools/configs_bench.sh ${@:-cfg2 cfg4 cfg5 cfg3}
