#!/usr/bin/env bash
# Short guarded GPU check: selected tests with a hard timeout, then C3 / C5 benches.
#   TAG=x TESTS_K="many_corners or paths" scripts/gpu_quick.sh
set -u
TAG=${TAG:-q}
mkdir -p gpurun_out
timeout ${TT:-300} python -m pytest tests -m gpu -x -q ${TESTS_K:+-k "$TESTS_K"} > gpurun_out/pytest_gpu_${TAG}.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_${TAG}.log
tail -3 gpurun_out/pytest_gpu_${TAG}.log
for cfg in ${CFGS:-c3_superblue}; do
  timeout ${BT:-180} python bench.py --config $cfg --quick --phases --steps 30 > gpurun_out/bench_${TAG}_${cfg}.json 2> gpurun_out/bench_${TAG}_${cfg}.err
  echo "$cfg rc=$?"; tail -c 600 gpurun_out/bench_${TAG}_${cfg}.json
done
