#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r2n.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r2n.log
tail -3 gpurun_out/pytest_gpu_r2n.log
TAG=r2n VARIANTS="base:;tcold:-DSTA_TC_THREADS=256 -DSTA_TC_TILE=2048" CFGS="c3_superblue c5_multicorner" bash scripts/gpu_variants.sh
