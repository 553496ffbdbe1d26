#!/usr/bin/env bash
# GPU parity tests (without the slow full-size C5 test) then a variant sweep.
#   TAG=r2i VARIANTS="base:;x:-DFOO=1" scripts/gpu_testvar.sh
set -u
TAG=${TAG:-r2}
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build_${TAG}.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -k "not c5_multicorner_full" > gpurun_out/pytest_gpu_${TAG}.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_${TAG}.log
tail -3 gpurun_out/pytest_gpu_${TAG}.log
bash scripts/gpu_variants.sh
