#!/usr/bin/env bash
# Round deliverables on one GPU box: build, GPU tests, smoke, the default bench
# line, reference arm, ncu launch list + full captures of the dominant kernels.
set -u
T=${T:-final}
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build_$T.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_$T.log
timeout 900 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$T.csv python bench.py --steps 3 --warmup 3 --quick > gpurun_out/ncu_launch_$T.log 2>&1
for K in fwd_persistent bwd_persistent rc_warp tc_persistent; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${K} \
    --launch-skip 3 --launch-count 1 -o gpurun_out/prof_${T}_${K} \
    python bench.py --steps 1 --warmup 3 --quick > gpurun_out/ncu_${K}_$T.log 2>&1
done
