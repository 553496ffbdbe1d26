set -u
mkdir -p gpurun_out
T=${T:-x}
python -m paper_2511_11660_b200.build --force > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${T}.csv python bench.py --steps 3 --warmup 3 --quick > gpurun_out/ncu_launch_${T}.log 2>&1
for K in rc_warp tc_persistent rc_block; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${K} \
    --launch-skip 3 --launch-count 1 -o gpurun_out/prof_${T}_${K} \
    python bench.py --steps 1 --warmup 3 --quick > gpurun_out/ncu_${K}_${T}.log 2>&1
done
