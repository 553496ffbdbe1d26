#!/usr/bin/env bash
# One gpurun call: build, GPU tests (TESTS=1), one bench line per build-flag
# set in NBS (comma-separated nvcc -D flags per set), and an STA_TRACE
# timeline of the default build.   T=tag NBS="-DSTA_FWD_BLOCKS=4 ..." bash scripts/gpu_sweep.sh
set -u
mkdir -p gpurun_out
T=${T:-x}
python __graft_entry__.py > gpurun_out/build_$T.log 2>&1
if [ "${TESTS:-1}" = 1 ]; then
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_$T.log
fi
for nb in ${NBS:-4}; do
  STA_NVCC_FLAGS="${nb//,/ }" python -m paper_2511_11660_b200.build --force > /dev/null 2>&1
  timeout 300 python bench.py --steps 20 --no-cpu-baseline > gpurun_out/bench_${T}_$(echo $nb | tr -dc "0-9_").json 2> gpurun_out/bench_${T}_$(echo $nb | tr -dc "0-9_").err
done
python -m paper_2511_11660_b200.build --force > /dev/null 2>&1
STA_TRACE_W=${TW:-5920,3552} timeout 300 python scripts/trace_run.py c3_superblue /tmp/trace_$T.csv > gpurun_out/trace_$T.txt 2>&1
du -sh gpurun_out/* | sort -h | tail -3
