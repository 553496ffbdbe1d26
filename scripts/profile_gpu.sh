#!/usr/bin/env bash
# Run on the GPU box (gpurun): launch list of one bench step (no graph, so
# every kernel is listed) + full ncu captures of selected kernels.
#   TAG=r1x ./scripts/profile_gpu.sh "fwd_stage:3 fwd_stage:60 bwd_stage:2 rc_tierC:0"
set -u
mkdir -p gpurun_out
TAG=${TAG:-r1}
STA_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 1 --warmup 0 --quick > gpurun_out/ncu_bench_${TAG}.log 2>&1
for spec in ${1:-"fwd_stage:3 bwd_stage:70"}; do
  K=${spec%%:*}; S=${spec##*:}
  STA_NO_GRAPH=1 ncu --set full --clock-control none --import-source on -k regex:${K} \
      --launch-skip ${S} --launch-count 1 -o gpurun_out/prof_${TAG}_${K}_${S} \
      python bench.py --steps 1 --warmup 0 --quick > gpurun_out/ncu_${K}_${S}_${TAG}.log 2>&1
done
