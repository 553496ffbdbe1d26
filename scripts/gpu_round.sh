#!/usr/bin/env bash
# One gpurun call: GPU parity tests, bench line, ncu launch list, full ncu
# captures of the two persistent propagation kernels.   TAG=r1b scripts/gpu_round.sh
set -u
TAG=${TAG:-r1}
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build_${TAG}.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
if [ "${NCU:-1}" = 1 ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 3 --warmup 3 --quick > gpurun_out/ncu_launch_${TAG}.log 2>&1
for K in fwd_persistent bwd_persistent; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${K} \
    --launch-skip 3 --launch-count 1 -o gpurun_out/prof_${TAG}_${K} \
    python bench.py --steps 1 --warmup 3 --quick > gpurun_out/ncu_${K}_${TAG}.log 2>&1
done
fi
