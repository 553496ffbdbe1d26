#!/usr/bin/env bash
# ncu evidence for one config: launch list (cold, serialised) and optional
# full captures.   TAG=r2b CFG=c3_superblue FULL="fwd_persistent bwd_persistent" scripts/gpu_prof.sh
set -u
TAG=${TAG:-r2}; CFG=${CFG:-c3_superblue}
mkdir -p gpurun_out
python -m paper_2511_11660_b200.build > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --config ${CFG} --steps 3 --warmup 3 --quick \
    > gpurun_out/ncu_launch_${TAG}.log 2>&1
for K in ${FULL:-}; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${K} \
    --launch-skip ${SKIP:-3} --launch-count 1 -o gpurun_out/prof_${TAG}_${K} \
    python bench.py --config ${CFG} --steps 1 --warmup 3 --quick > gpurun_out/ncu_${K}_${TAG}.log 2>&1
done
