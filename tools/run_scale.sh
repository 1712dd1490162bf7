#!/bin/bash
# Multi-GPU bench lines (run under `gpurun --gpus N`): N=1 plain, then torchrun
# for every power of two up to the visible GPU count.
#   tools/run_scale.sh <workload> <steps> [tag]
set -u
WL=${1:-c3}; STEPS=${2:-5}; TAG=${3:-$WL}
mkdir -p gpurun_out
NG=$(python -c "import torch; print(torch.cuda.device_count())")
python bench.py --workload $WL --steps $STEPS --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/scale_${TAG}_n1.json 2> gpurun_out/scale_${TAG}_n1.err
n=2
while [ $n -le $NG ]; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + n)) \
    bench.py --gpus $n --workload $WL --steps $STEPS --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/scale_${TAG}_n$n.json 2> gpurun_out/scale_${TAG}_n$n.err
  n=$((n * 2))
done
for f in gpurun_out/scale_${TAG}_n*.json; do echo "$f $(tail -c 400 $f)"; done
