#!/usr/bin/env bash
# One gpurun call: build, GPU parity tests, smoke, bench line (optional C5 bench).
#   TAG=r2a scripts/gpu_check.sh
set -u
TAG=${TAG:-r2}
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build_${TAG}.log 2>&1
timeout ${PYTEST_TIMEOUT:-1500} python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_${TAG}.log
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
if [ "${C5:-0}" = 1 ]; then
timeout 900 python bench.py --config c5_multicorner --no-cpu-baseline > gpurun_out/bench_c5_${TAG}.json 2> gpurun_out/bench_c5_${TAG}.err
fi
